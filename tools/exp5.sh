cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
for d in 1 2 3 4; do echo "chunk_div=$d"; GBNR_CHUNK_DIV=$d timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2; done
for f in 0.5 0.6; do echo "chunk_div=3 stage=$f"; GBNR_STAGE_FRAC=$f GBNR_CHUNK_DIV=3 timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2; done

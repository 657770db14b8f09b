cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for sf in 0.4 0.5 0.6; do echo "stage_frac=$sf"; GBNR_STAGE_FRAC=$sf timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2; done

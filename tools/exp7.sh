cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for a in 0 4 8 16 32; do echo "l2_ahead=$a"; GBNR_L2_AHEAD=$a timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2; done

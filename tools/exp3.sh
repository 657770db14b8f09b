cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for o in "$@"; do timeout 300 python tools/gpu_quick.py synth9241 10000 $o 2>&1 | tail -2; done

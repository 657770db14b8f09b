cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for tl in 0 1 2 3; do echo "team_levels=$tl"; GBNR_TEAM_LEVELS=$tl timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "montecarlo and synth9241 or invariance" 2>&1 | tail -1; GBNR_TEAM_LEVELS=$tl timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2; done

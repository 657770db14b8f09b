#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small parity cases: gpu_sanitize.sh TAG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-dev}
mkdir -p $O
make -s >/dev/null 2>&1
# Monte-Carlo parity on small grids (full-width tiles, backward-walk pair records) and
# the tile-width invariance test at widths 8 and 14 (lanes shadowing, generic kernels)
SEL='(montecarlo and (case14 or synth118 or synth300)) or (tile_width and (8 or 14))'
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" > $O/${T}_memcheck.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" > $O/${T}_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --num-cuda-barriers 200000 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" > $O/${T}_synccheck.log 2>&1
grep -h "SUMMARY\|passed\|failed" $O/${T}_*check.log

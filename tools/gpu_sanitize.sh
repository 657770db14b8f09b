#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small parity cases: gpu_sanitize.sh TAG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-dev}
mkdir -p $O
make -s >/dev/null 2>&1
# Monte-Carlo parity on small grids (full-width tiles, backward-walk pair records) and
# the tile-width invariance test at widths 8 and 14 (lanes shadowing, generic kernels)
FULL='montecarlo and (case14 or synth118 or synth300)'
SEL="($FULL) or (tile_width and (8 or 14))"
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" > $O/${T}_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --num-cuda-barriers 200000 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" > $O/${T}_synccheck.log 2>&1
# racecheck: full-width tiles must be hazard-free; at narrower widths the shadow
# lanes (>= tile width) repeat lane width-1's shared-memory stores of the same
# values in the same warp instruction, which racecheck reports as warnings
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$FULL" > $O/${T}_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tile_width and (8 or 14)" > $O/${T}_racecheck_narrow.log 2>&1
grep -h "SUMMARY\|passed\|failed" $O/${T}_*check*.log

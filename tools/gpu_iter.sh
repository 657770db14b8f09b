#!/bin/bash
# Development pass on the GPU box: parity tests, then per-kernel timings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
make -s 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -30 $O/pytest_gpu.log
for c in ${QUICK:-"synth9241 10000"}; do timeout 300 python tools/gpu_quick.py $c $QOPTS 2>&1 | tail -5; done

#!/bin/bash
# Round-2 GPU pass: parity tests, quick per-kernel timings (headline + stress grid), bench.
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-r02}
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/host.txt; lscpu >> $O/host.txt
make -s 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$T.log
for c in ${QUICK:-synth9241 synth9241x}; do timeout 300 python tools/gpu_quick.py $c 10000 >> $O/quick_$T.log 2>&1; done
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_$T.log 2>&1

#!/bin/bash
# One GPU-box pass: parity tests, quick per-kernel timings, bench, ncu launch list.
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/host.txt; lscpu >> $O/host.txt
make -s 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/gpu_quick.py synth9241 10000 > $O/quick9241.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_one.py synth9241 10000 > $O/ncu_launch.log 2>&1

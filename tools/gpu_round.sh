#!/bin/bash
# Round evidence on the GPU box: parity tests, bench, ncu launch list, per-kernel
# DRAM bytes, --set full captures of the walk kernels.  Usage: gpu_round.sh TAG
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-r01}
mkdir -p $O
make -s 2>&1 | tail -3
nproc > $O/host.txt; lscpu >> $O/host.txt; nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$T.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/dram_$T.csv python tools/prof_one.py synth9241 10000 > $O/ncu_dram_$T.log 2>&1
for K in ${KERNELS:-lu_walk_kernel bs_walk_kernel jacobian_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip ${SKIP:-1} --launch-count 1 \
     -o $O/full_${T}_$K -f python tools/prof_one.py synth9241 10000 > $O/ncu_full_${T}_$K.log 2>&1
done
ls -la $O

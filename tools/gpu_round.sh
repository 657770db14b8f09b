#!/bin/bash
# One GPU-box evidence pass: parity tests, quick per-kernel timings (headline + stress grid),
# bench, ncu launch list / DRAM bytes / --set full of the walk kernels.
#   gpu_round.sh TAG   (env: PYTEST_K selects tests, SKIP_NCU=1, SKIP_TESTS=1, QUICK="cases")
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-r02}
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/host.txt; lscpu >> $O/host.txt; free -g >> $O/host.txt
make -s 2>&1 | tail -3
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$T.log
fi
for c in ${QUICK:-synth9241 synth9241x}; do timeout 300 python tools/gpu_quick.py $c 10000 >> $O/quick_$T.log 2>&1; done
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_$T.log 2>&1
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$T.csv \
      python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 1 > $O/ncu_launch_$T.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $O/dram_$T.csv python tools/prof_one.py synth9241 10000 > $O/ncu_dram_$T.log 2>&1
  for K in ${KERNELS:-lu_walk_kernel bs_walk_kernel}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip ${SKIP:-1} --launch-count 1 \
       -o $O/full_${T}_$K -f python tools/prof_one.py synth9241 10000 > $O/ncu_full_${T}_$K.log 2>&1
  done
fi
ls -la $O

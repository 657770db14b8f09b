#!/bin/bash
# ncu captures for profiles/: per-kernel DRAM bytes of one full solve (every
# launch) and `--set full` reports of the top kernels.  Usage: gpu_ncu.sh TAG
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-r01}
mkdir -p $O
make -s 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/dram_$T.csv python tools/prof_one.py synth9241 10000 > $O/ncu_dram_$T.log 2>&1
for K in ${KERNELS:-lu_pipe_kernel lu_level_kernel tri_pipe_kernel jacobian_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip ${SKIP:-2} --launch-count 1 \
     -o $O/full_${T}_$K -f python tools/prof_one.py synth9241 10000 > $O/ncu_full_${T}_$K.log 2>&1
done
ls -la $O

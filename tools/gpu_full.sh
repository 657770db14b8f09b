#!/bin/bash
# --set full captures only (development): gpu_full.sh TAG  (KERNELS, SKIP env)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-dev}
mkdir -p $O
make -s 2>&1 | tail -3
for K in ${KERNELS:-lu_walk_kernel bs_walk_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip ${SKIP:-1} --launch-count 1 \
     -o $O/full_${T}_$K -f python tools/prof_one.py synth9241 10000 > $O/ncu_full_${T}_$K.log 2>&1
done
ls -la $O | grep $T

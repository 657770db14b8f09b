#!/bin/bash
# Walker time breakdown (GBNR_PROF build) and the shared-memory / CTA sweep of the
# LU walk.  usage: gpu_prof.sh TAG
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-prof}
mkdir -p $O
make -s 2>&1 | tail -3
make -s prof 2>&1 | tail -3
for N in ${TASKS:-2500 10000}; do
  GBNR_LIB=$PWD/paper_2101_02270_b200/libgbnr_prof.so GBNR_DBG=8 timeout 300 python tools/gpu_quick.py synth9241 $N >> $O/prof_$T.log 2>&1
done
TASKS="2500 5000 10000" bash tools/smem_sweep.sh >> $O/smem_sweep_$T.log 2>&1

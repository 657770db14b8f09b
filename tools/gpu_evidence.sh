#!/bin/bash
# Round-end evidence on one box: gpu_round.sh (tests, quick timings, bench, ncu) +
# BASELINE configs + the reference arm + a 2-rank bench on one GPU + sanitizers.
#   gpu_evidence.sh TAG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; T=${1:-r02}
mkdir -p $O
KERNELS="${KERNELS:-lu_walk_kernel bs_walk_kernel npm_kernel vupdate_kernel}" bash tools/gpu_round.sh $T > $O/round_$T.log 2>&1
timeout 1200 python tools/bench_configs.py $O/configs_$T.json > $O/configs_$T.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference_$T.log 2>&1
GBNR_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --tasks 5000 --steps 3 --warmup 3 --no-cpu > $O/bench2_$T.log 2>&1
bash tools/gpu_sanitize.sh $T > $O/sanitize_$T.txt 2>&1
tail -3 $O/pytest_gpu_$T.log; tail -1 $O/bench_$T.log; cat $O/sanitize_$T.txt

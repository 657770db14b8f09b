cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
for i in 1 2; do
echo "A (head)"; GBNR_LIB=$PWD/gpurun_ab_head.so timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2
echo "B (work)"; timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2
done

cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
for T in 2500 5000 10000 14000; do timeout 300 python tools/gpu_quick.py synth9241 $T 2>&1 | tail -2; done

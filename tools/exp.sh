cd $GRAFT_REPO_ROOT; make -s >/dev/null 2>&1
for d in 0 1 2 3; do echo "DBG=$d"; GBNR_DBG=$d timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2; done

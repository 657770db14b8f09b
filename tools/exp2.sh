cd "$GRAFT_REPO_ROOT"; make -s >/dev/null 2>&1
GBNR_DBG=4 timeout 300 python tools/prof_one.py synth9241 10000 2>&1 | grep walk | head -60

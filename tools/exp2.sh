cd "$GRAFT_REPO_ROOT"; touch paper_2101_02270_b200/csrc/kernels.cu; make -s GBNR_TRACE=1 >/dev/null 2>&1
GBNR_DBG=4 timeout 300 python tools/prof_one.py synth9241 10000 2>&1 | grep "walk] tile 0 " | head -400

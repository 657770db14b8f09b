#!/bin/bash
# Tile-width sweep of one solve (GBNR_TW forces the width; auto = the plan's choice).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for T in ${TASKS:-10000}; do
  for tw in ${TWS:-auto 32 24 16}; do
    echo -n "tw=$tw "
    if [ "$tw" = auto ]; then timeout 300 python tools/gpu_quick.py ${CASE:-synth9241} $T 2>&1 | head -1
    else GBNR_TW=$tw timeout 300 python tools/gpu_quick.py ${CASE:-synth9241} $T 2>&1 | head -1; fi
  done
done

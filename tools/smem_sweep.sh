#!/bin/bash
# Per-tile latency vs shared-memory pool: LU walk time at fixed tasks for
# several CTA budgets (GBNR_SMEM_BUDGET bytes, GBNR_CTAS resident CTAs per SM).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for T in ${TASKS:-5000 10000}; do
  for cfg in "76800 3" "113000 2" "150000 1" "225000 1"; do
    set -- $cfg
    echo -n "budget=$1 ctas=$2 "
    GBNR_SMEM_BUDGET=$1 GBNR_CTAS=$2 timeout 300 python tools/gpu_quick.py synth9241 $T 2>&1 | head -1
  done
done

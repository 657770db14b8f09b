#!/bin/bash
# A/B the prebuilt library variants on one box: ab.sh LIB1 LIB2 ... (ROUNDS env, default 2)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for r in $(seq ${ROUNDS:-2}); do
  for L in "$@"; do
    echo -n "$L: "; GBNR_LIB=$PWD/$L timeout 300 python tools/gpu_quick.py synth9241 10000 2>&1 | tail -2 | head -1
  done
done

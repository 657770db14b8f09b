#!/bin/bash
# Parameter sweep on one box: each argument is "ENV=.. ENV=.. -- key=val ..." (quoted)
#   sweep.sh "GBNR_STAGE_FRAC=0.3 --" "-- prefetch=4"
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
make -s >/dev/null 2>&1
for cfg in "$@"; do
  envs="${cfg%%--*}"; opts="${cfg#*--}"
  echo -n "[$cfg] "
  env $envs timeout 300 python tools/gpu_quick.py synth9241 ${TASKS:-10000} $opts 2>&1 | tail -2 | head -1
done

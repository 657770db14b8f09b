#!/bin/bash
# Experiment sweep on the GPU box: parity tests, then per-config timings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
make -s >/dev/null 2>&1 || make
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for o in "$@"; do timeout 300 python tools/gpu_quick.py synth9241 10000 $o 2>&1 | tail -2; done

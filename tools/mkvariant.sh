#!/bin/bash
# Build a library variant from a patch script without touching the tree:
#   mkvariant.sh NAME PATCH.py   -> ab/NAME.so   (PATCH.py edits kernels.cu in place)
set -e
cd /root/repo
K=paper_2101_02270_b200/csrc/kernels.cu
cp $K /tmp/_k_orig.cu
python "$2" $K
make -s 2>&1 | grep -E "error" && { cp /tmp/_k_orig.cu $K; exit 1; }
cp paper_2101_02270_b200/libgbnr.so ab/$1.so
cp /tmp/_k_orig.cu $K
make -s

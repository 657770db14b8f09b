#!/bin/bash
# Build a library variant from a patch script without touching the tree:
#   mkvariant.sh NAME PATCH.py  -> ab/NAME.so  (PATCH.py gets kernels.cu's path and may
#   edit any file under csrc/; the directory is restored afterwards)
set -e
cd /root/repo
C=paper_2101_02270_b200/csrc
rm -rf /tmp/_csrc_orig; cp -r $C /tmp/_csrc_orig
python "$2" $C/kernels.cu
if make -s 2>&1 | grep -E "error"; then rm -rf $C; cp -r /tmp/_csrc_orig $C; exit 1; fi
cp paper_2101_02270_b200/libgbnr.so ab/$1.so
rm -rf $C; cp -r /tmp/_csrc_orig $C
touch $C/*.cu $C/*.cpp
make -s

#!/bin/bash
# build a scratch variant of libhm_b200.so: mkscratch.sh <name> <nvflags>
set -e
name=$1; shift
d=/root/repo/scratch/$name
rm -rf $d; mkdir -p $d
cp -r /root/repo/paper_2605_25092_b200/csrc $d/csrc
rm -rf $d/csrc/build
make -s -j8 -C $d/csrc LIB=$d/lib INC="-I/root/repo/include -Ikernels" HM_EXTRA_NVFLAGS="$*" HM_EXTRA_CXXFLAGS="$*" $d/lib/libhm_b200.so 2>&1 | grep -i error || true
cp /root/repo/paper_2605_25092_b200/lib/libhm_synth.so $d/lib/
ls -la $d/lib

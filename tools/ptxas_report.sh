#!/bin/bash
# Per-variant register / spill report from ptxas -v (run from anywhere; rebuilds the variant TUs).
cd "$(dirname "$0")/../paper_1510_04995_b200/csrc"
for f in variants_const7 variants_var7 variants_const25 variants_var25; do
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
     -I. -I../../include -Xptxas -v -c $f.cu -o /tmp/$f.o 2>&1 |
  awk '/Compiling entry function/ {n=$0; sub(/.*zwave_kernelILi/,"",n); name=n}
       /spill stores/ {sp=$5" st/"$9" ld"}
       /Used [0-9]+ registers/ {print name, $5" regs", sp}' | c++filt | sed 's/_ZN9girih_gpu12//'
done

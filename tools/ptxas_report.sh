#!/bin/bash
# Per-kernel register / spill report from ptxas -v:  tools/ptxas_report.sh variants_var7.cu
# (template arguments: KIND, TB, LX, LY, NT, P, PA, MINB, CHAIN, CF = cy | flags << 8, INSTR)
cd "$(dirname "$0")/../paper_1510_04995_b200/csrc"
f=${1:-variants_var7.cu}
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -I. -I../../include -Xptxas -v -c $f -o /tmp/x.o 2>&1 | awk '/Compiling entry function/{n=$0; sub(/.*function ./,"",n); sub(/. for .*/,"",n)} /spill stores/{sp=$5"/"$9} /Used [0-9]+ registers/{print n, "regs="$5, "spill="sp}' | while read n r s; do echo "$(echo $n | c++filt | sed 's/.*zwave_kernel<\([^>]*\)>.*/\1/') $r $s"; done

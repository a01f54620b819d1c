#!/bin/bash
# registers / spills per kernel of one .cu (ptxas -v), filtered by a pattern
f=$1; pat=$2
cd "$(dirname "$0")/../paper_1812_07625_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xptxas -v -c $f -o /tmp/regs.o 2>&1 | \
  awk -v pat="$pat" '/Compiling entry function/ {name=$0; sub(/.*function ./,"",name); sub(/. for.*/,"",name)} /Used/ && name ~ pat {print name; print "   " $0} /spill/ && name ~ pat {print "   " $0}' | c++filt | grep -v "^$"

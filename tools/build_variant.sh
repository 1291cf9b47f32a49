#!/bin/bash
# usage: tools/build_variant.sh <name> [-DKNOB=VALUE ...]
# Experiment build: sweep_march2.cu alone, restricted to the production kernel pairs
# (MB4_QUICK_PAIRS: first-sweep depth 6, later depths 1 and 2), linked with the other
# objects of the last full libmb4cu.so build -> paper_2003_04345_b200/lib_<name>.so
# (select it with MB4CU_LIB=...; tools/variants.sh compares several on the GPU box).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
obj=build/lib_${name}.so.sweep_march2.cu.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 \
  -DMB4_QUICK_PAIRS "$@" -I include -I build/gen -Xptxas -v \
  -c paper_2003_04345_b200/csrc/sweep_march2.cu -o $obj 2> build/lib_${name}.ptxas.log
others=$(ls build/libmb4cu.so.*.o | grep -v sweep_march2)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2003_04345_b200/lib_${name}.so $obj $others -lcudart -lcufft -lpthread -ldl
# registers / spills of the production launches
python3 - "$name" <<'PY'
import re, sys
log = open(f"build/lib_{sys.argv[1]}.ptxas.log").read()
for m in re.finditer(r"Compiling entry function '(\S+)'.*?\n.*?\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n.*?Used (\d+) registers", log):
    name = m.group(1)
    k = re.search(r"kernelILi(\d)ELi(\d)ELi(\d+)ELb(\d)ELb(\d)ELb(\d)ELi(\d)E", name)
    if k and k.group(4) == "1" and k.group(6) == "1" and k.group(7) in "12" and k.group(5) == "0":
        print("MF,M,NT,ISO,GHOST,DEF,PH =", ",".join(k.groups()), "regs", m.group(5), "spill st/ld", m.group(3), m.group(4))
PY

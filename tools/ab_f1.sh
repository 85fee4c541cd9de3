#!/bin/bash
# F1-only timing (tools/time_f1.py) of library variants.  usage: tools/ab_f1.sh [N m] -- v1 v2 ...
N=128; M=10
if [ "$3" = "--" ]; then N=$1; M=$2; shift 3; fi
for v in "$@"; do
  if [ "$v" = main ]; then unset B2L_LIB_PATH; else export B2L_LIB_PATH=$PWD/scratch/variants/$v.so; fi
  echo -n "$v: "; python tools/time_f1.py $N $M 2>&1 | tail -1
done

#!/bin/bash
# A/B of library variants (tools/build_variant.py): C2 step medians and the
# per-kernel timer pass for each variant.  usage: tools/ab.sh name1 name2 ...
# ("main" = the in-tree library).  Diagnostic only.
for v in "$@"; do
  if [ "$v" = main ]; then unset B2L_LIB_PATH; else export B2L_LIB_PATH=$PWD/scratch/variants/$v.so; fi
  echo "=== $v"
  python tools/step_times.py 128 10 120 2>&1 | tail -2
  python tools/time_config.py 128 10 2>&1 | tail -4
done

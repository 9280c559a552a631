#!/usr/bin/env bash
# Interleaved A/B timing of prefill variants (tools/bin/libmoa_<name>.so, tools/build_variant.py):
#   bash tools/ab_prefill.sh "C2 8 0" REPS name1 name2 ...     (name "main" = the in-tree build)
ARGS=$1; REPS=$2; shift 2
for r in $(seq 1 $REPS); do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=paper_2406_14909_b200/libmoa.so; else lib=tools/bin/libmoa_$v.so; fi
    echo -n "$v: "; MOA_LIB=$lib timeout 300 python tools/time_prefill.py $ARGS 2>&1 | tail -1
  done
done

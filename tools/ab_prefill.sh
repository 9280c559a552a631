#!/usr/bin/env bash
# Interleaved A/B timing of prefill variants (tools/bin/libmoa_<name>.so, tools/build_variant.py):
#   bash tools/ab_prefill.sh "C2 8 0" REPS name1 name2 ...     (name "main" = the in-tree build, "cluster" = it with MOA_PP_CLUSTER=1)
ARGS=$1; REPS=$2; shift 2
for r in $(seq 1 $REPS); do
  for v in "$@"; do
    env=""
    if [ "$v" = main ]; then lib=paper_2406_14909_b200/libmoa.so;
    elif [ "$v" = cluster ]; then lib=paper_2406_14909_b200/libmoa.so; env="MOA_PP_CLUSTER=1";
    elif [ "$v" = nosched ]; then lib=paper_2406_14909_b200/libmoa.so; env="MOA_PP_SCHED=0";
    elif [ "${v#cost}" != "$v" ]; then lib=paper_2406_14909_b200/libmoa.so; env="MOA_PP_SCHED_COST=${v#cost}";
    else lib=tools/bin/libmoa_$v.so; fi
    echo -n "$v: "; env $env MOA_LIB=$lib timeout 300 python tools/time_prefill.py $ARGS 2>&1 | tail -1
  done
done

#!/usr/bin/env bash
# Profiling pass for one round (run on the GPU box from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash tools/profile_round.sh r01'
# Writes gpurun_out/<round>_*: the ncu launch list of the bench command, full ncu
# captures of the decode and prefill kernels and a clocks log.  tools/summarize_profiles.py
# turns them into the committed summaries under profiles/.
set -u
R=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
K='regex:prefill_pp_kernel|prefill_f32_kernel|decode_mma_kernel|decode_kernel|cache_fill_kernel|kv_append_kernel'
L=32; T=512
# warm-up launches of bench.py (--warmup 3): 3 steps x (L prefill with fused fill + T cross-layer decode)
SKIP=$((3 * (L + T)))

# 1) launch list of the same command bench.py runs (per-launch device time, serialised)
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s $SKIP -c 600 \
  --csv --log-file $OUT/${R}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > $OUT/${R}_launches_bench.log 2>&1
echo "launch list rc=$?"

# 2) full capture of the dominant kernel (decode) and of the prefill kernel
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 1 -c 1 \
  -o $OUT/${R}_decode_full python tools/prof_run.py layers --layers 32 --first-layer 0 --tokens 2 > $OUT/${R}_decode_full.log 2>&1
echo "decode full rc=$?"
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:prefill_pp -s 1 -c 1 \
  -o $OUT/${R}_prefill_full python tools/prof_run.py prefill --layers 2 > $OUT/${R}_prefill_full.log 2>&1
echo "prefill full rc=$?"
ls -la $OUT | grep "$R"

#!/usr/bin/env bash
# Per-config profiler captures on the GPU box (one GPU), written under gpurun_out/<tag>/:
#   1. the bench line of the config (no profiler) -> accepted steps per launch
#   2. the ncu launch list of a short bench run (cold-cache, serialised per-launch times)
#   3. one `ncu --set full` capture of the trace kernel, summarised into ncu_<cfg>_trace.json
# Usage: bash profiles/capture.sh <tag> <config> [<config> ...]
set -u
tag=$1; shift
out=gpurun_out/$tag
mkdir -p "$out"
for cfg in "$@"; do
  python bench.py --config "$cfg" --steps 3 --warmup 3 --no-e2e --no-cpu --no-driver \
    > "$out/bench_$cfg.json" 2> "$out/bench_$cfg.err" || { echo "bench $cfg failed"; continue; }
  steps=$(python -c "import json,sys; print(json.loads(open('$out/bench_$cfg.json').read().strip().splitlines()[-1])['accepted_steps_per_trace'])")
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$out/launches_$cfg.csv" \
    python bench.py --config "$cfg" --steps 2 --warmup 1 --no-e2e --no-cpu --no-driver \
    > "$out/launches_$cfg.log" 2>&1
  ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 \
    -o "$out/trace_$cfg" -f \
    python bench.py --config "$cfg" --steps 1 --warmup 1 --no-e2e --no-cpu --no-driver \
    > "$out/ncu_$cfg.log" 2>&1
  python profiles/summarize_ncu.py "$out/trace_$cfg.ncu-rep" "$out/ncu_${cfg}_trace.json" \
    "trace_kernel default, $cfg" \
    "python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu --no-driver" \
    "$steps" > "$out/summary_$cfg.txt" 2>&1
  echo "$cfg: steps=$steps $(head -c 300 "$out/summary_$cfg.txt" | tr '\n' ' ')"
  # reports are tens of MB: keep the summary only (gpurun copies back <= 64 MiB)
  [ "${KEEP_REP:-0}" = 1 ] || rm -f "$out/trace_$cfg.ncu-rep"
done

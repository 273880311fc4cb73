#!/usr/bin/env bash
# One `ncu --set full` capture of the trace kernel of `bench.py --config <cfg>` under an
# environment setting (e.g. PHG_BRICKS=1), summarised into gpurun_out/<tag>/ncu_<cfg>_<label>.json
# Usage: bash profiles/capture_env.sh <tag> <cfg> <label> <steps_per_launch> [VAR=value ...]
set -u
tag=$1; cfg=$2; label=$3; steps=$4; shift 4
out=gpurun_out/$tag; mkdir -p "$out"
env "$@" ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 1 -c 1 \
  -o "$out/trace_${cfg}_$label" -f \
  python bench.py --config "$cfg" --steps 1 --warmup 1 --no-e2e --no-cpu --no-driver \
  > "$out/ncu_${cfg}_$label.log" 2>&1
python profiles/summarize_ncu.py "$out/trace_${cfg}_$label.ncu-rep" "$out/ncu_${cfg}_${label}.json" \
  "trace_kernel $label, $cfg" "$* python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu --no-driver" \
  "$steps" > "$out/summary_${cfg}_$label.txt" 2>&1
head -c 400 "$out/summary_${cfg}_$label.txt"; echo
[ "${KEEP_REP:-0}" = 1 ] || rm -f "$out/trace_${cfg}_$label.ncu-rep"

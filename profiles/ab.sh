#!/usr/bin/env bash
# A/B of two library builds on the same box: alternates `python bench.py` runs of the current
# libphg_b200.so and the build at $1 (e.g. ab_old/libphg_b200.so), $3 rounds, config $2.
# Usage: bash profiles/ab.sh <other.so> <config> <rounds> <tag> [bench args...]
set -u
other=$1; cfg=$2; rounds=$3; tag=$4; shift 4
out=gpurun_out/$tag; mkdir -p "$out"
for r in $(seq 1 "$rounds"); do
  for which in new old; do
    if [ "$which" = old ]; then export PHG_LIB_PATH=$other; else unset PHG_LIB_PATH; fi
    python bench.py --config "$cfg" --steps 5 --warmup 3 --no-e2e --no-cpu --no-driver "$@" \
      > "$out/ab_${cfg}_${which}_$r.json" 2> "$out/ab_${cfg}_${which}_$r.err"
    python -c "import json;d=json.loads(open('$out/ab_${cfg}_${which}_$r.json').read().strip().splitlines()[-1]);print('$cfg $which $r', round(d['roofline']['kernel_ms'],3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  done
done

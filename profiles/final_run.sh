#!/usr/bin/env bash
# End-of-change measurement set on one GPU box, written under gpurun_out/<tag>/:
#   GPU tests (release + checked build), per-config ncu captures (capture.sh), the driver's
#   default commands for both arms, and full bench lines for every config.
# Usage: bash profiles/final_run.sh <tag> [--no-tests]
set -u
tag=$1; shift
out=gpurun_out/$tag; mkdir -p "$out"
if [ "${1:-}" != "--no-tests" ]; then
  python -m pytest tests -m gpu -q > "$out/gputest.log" 2>&1; tail -1 "$out/gputest.log"
  PHG_CHECKED_LIB=1 python -m pytest tests -m gpu -q > "$out/gputest_checked.log" 2>&1
  tail -1 "$out/gputest_checked.log"
fi
bash profiles/capture.sh "$tag" C3 C2 C5 C1 C3s > "$out/capture.log" 2>&1; cat "$out/capture.log" | cut -c1-160
python bench.py > "$out/final_default_bench.jsonl" 2> "$out/final_default_bench.err"
python bench.py --impl reference > "$out/final_default_ref.jsonl" 2> "$out/final_default_ref.err"
for c in C1 C2 C3 C3s C5 C4; do
  python bench.py --config $c --steps 10 --warmup 3 > "$out/final_bench_$c.jsonl" 2> "$out/final_bench_$c.err"
done
python - "$out" <<'PY'
import json, sys, glob, os
for f in sorted(glob.glob(os.path.join(sys.argv[1], "final_*.jsonl"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), "ERR", e); continue
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(os.path.basename(f), d.get("config", {}).get("workload", "")[:4], "value %.3g" % d["value"],
          "csr %.3g" % (d.get("value_csr") or 0), "kern", r.get("kernel_ms"), "frac", r.get("frac"),
          "e2e %.3g" % (e.get("value") or 0), (d.get("trace_kernel") or {}).get("variant"))
PY

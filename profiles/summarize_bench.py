"""One line per bench record: value, value_csr, K1 ms, roofline frac, DRAM B/step, e2e and
the CPU legs.  Usage: summarize_bench.py <file.jsonl> ..."""
import json
import os
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "ERR", e)
        continue
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    cb = d.get("cpu_baseline") or {}
    hb = (r.get("hbm") or {})
    print(f"{os.path.basename(f):28s} {d.get('config', {}).get('workload', '')[:4]:5s}"
          f" value {d['value'] / 1e9:7.3f}G csr {(d.get('value_csr') or 0) / 1e9:6.2f}G"
          f" ms {d.get('ms_per_step', 0):7.3f} K1 {r.get('kernel_ms') or 0:7.3f}"
          f" frac {r.get('frac') or 0:.3f} dramB {hb.get('dram_bytes_per_step') or 0:5.1f}"
          f" e2e {(e.get('value') or 0) / 1e9:5.2f}G cpu {(cb.get('value') or 0) / 1e6:6.2f}M"
          f" init {((cb.get('init_guide_strands') or {}).get('value') or 0) / 1e6:5.2f}M"
          f" one {((cb.get('one_core') or {}).get('value') or 0) / 1e6:5.2f}M"
          f" clk {(d.get('clocks') or {}).get('sm_mhz')} {(d.get('clocks') or {}).get('reasons')}")

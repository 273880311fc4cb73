"""Per-instruction execution counts and stall samples from an `ncu --page source --csv
--print-source sass` export: writes an annotated listing (executions per accepted step) and
prints the opcode mix.  Usage: annotate_source.py <source_sass.csv> <steps> <out.txt>"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2])
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ith = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
ismp = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iex]) for r in data)
samples = sum(int(r[ismp]) for r in data)
mix, stall = {}, {}
with open(sys.argv[3], "w") as out:
    for r in data:
        ex, th, sm = int(r[iex]), int(r[ith]), int(r[ismp])
        src = r[isrc].strip()
        out.write(f"{r[ia][-5:]} {ex * 32 / steps:7.3f} {th / steps:7.3f} {sm:6d}  {src}\n")
        t = src.split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
        mix[op] = mix.get(op, 0) + ex * 32 / steps
        stall[op] = stall.get(op, 0) + sm
print(f"warp-inst per step (x32): {tot * 32 / steps:.1f}; stall samples {samples}")
for op, v in sorted(mix.items(), key=lambda x: -x[1])[:30]:
    print(f"{op:10s} {v:7.1f}  {stall[op] / max(samples, 1):.3f}")

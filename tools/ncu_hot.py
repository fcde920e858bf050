"""Per-instruction hot spots from an ncu source page (SASS): instruction and stall-sample shares."""
import csv, sys, subprocess, re
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, isamp, iexe = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[iexe].isdigit(): continue
    data.append((r[ia], r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0)))
T = sum(d[3] for d in data); S = sum(d[2] for d in data)
print(f"total inst {T:.3e}, samples {S}")
# opcode mix
mix = {}
for a, s, smp, e in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0] if s else "?"
    mix[op] = mix.get(op, 0) + e
for op, e in sorted(mix.items(), key=lambda x: -x[1])[:25]:
    print(f"  {op:28s} {100*e/T:5.1f}%")
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    for a, s, smp, e in data:
        off = int(a, 16) - int(data[0][0], 16)
        if lo <= off <= hi:
            print(f"{off:05x} {e:12d} {smp:6d}  {s[:70]}")

"""Per-CUDA-line instruction and stall-sample shares from an ncu report (cuda,sass view).

    python tools/ncu_lines.py <report.ncu-rep> <kernel regex> [top]
"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
fname, cur, hdr = "?", None, None
agg = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:90])
    if cur is None:
        continue
    e = r[ie].strip()
    s = r[isamp].strip()
    a = agg.setdefault(cur, [0, 0])
    a[0] += int(e) if e.isdigit() else 0
    a[1] += int(s) if s.isdigit() else 0
T = sum(v[0] for v in agg.values()) or 1
S = sum(v[1] for v in agg.values()) or 1
print(f"total inst {T:.3e}  samples {S}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:14s}{k[1]:5d} {100 * v[0] / T:5.1f}% inst {100 * v[1] / S:5.1f}% smp  {k[2]}")

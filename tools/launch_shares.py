"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[1:]:
    if r[iv].replace(",", "").replace(".", "").isdigit():
        name = r[ik].split("<")[0].split("(")[0].replace("void ", "").replace("ente::", "")
        v = float(r[iv].replace(",", "")) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[r[iu]]
        tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':28s} {'launches':>8s} {'ms':>10s} {'share':>7s}   (ncu: cold-cache, serialised)")
for k, v in tot.most_common():
    print(f"{k:28s} {cnt[k]:8d} {v:10.3f} {100*v/T:6.1f}%")
print(f"{'total':28s} {sum(cnt.values()):8d} {T:10.3f}")

"""Summarise an ncu --set full report (raw page) for the sweep kernels."""
import csv, subprocess, sys
KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]
STALL = "smsp__average_warps_issue_stalled_"
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
if "--traffic" in sys.argv:  # {kernel: dram read+write bytes per launch} for bench.py
    import json
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("<")[0].replace("void ", "").split("(")[0].strip().split("::")[-1]
        # launch labels of bench.py's kernel profile (the compacted kNN sweep is "knn_pass")
        name = {"knn_pass_kernel": "knn_pass", "knn_compact_kernel": "knn_pass",
                "count_pass_kernel": "count_pass", "count_pass_direct_kernel": "count_pass"}.get(name, name)
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1)
        res.setdefault(name, tot)
    if "--merge" in sys.argv:  # --merge <traffic.json> --config <C>: res under that config key
        path = sys.argv[sys.argv.index("--merge") + 1]
        cfg = sys.argv[sys.argv.index("--config") + 1]
        try:
            cur = json.load(open(path))
        except OSError:
            cur = {}
        cur.setdefault(cfg, {}).update(res)
        cur[cfg]["_capture"] = sys.argv[1]
        json.dump(cur, open(path, "w"), indent=1)
    print(json.dumps(res))
    sys.exit(0)
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d["Kernel Name"][:70])
    for k in KEYS:
        if k in d: print(f"   {k:70s} {d[k]} {units[hdr.index(k)]}")
    st = sorted(((float(d[k] or 0), k) for k in hdr if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")), reverse=True)[:8]
    for v, k in st:
        print(f"   stall {k[len(STALL):-len('_per_issue_active.ratio')]:30s} {v:.3f}")

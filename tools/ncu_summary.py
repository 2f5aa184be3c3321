"""Summarise ncu outputs into profiles/:
  launches.csv (gpu__time_duration per launch) -> per-kernel totals and shares
  <name>.ncu-rep (--set full)                -> duration, DRAM bytes, throughputs
usage: python tools/ncu_summary.py <launches.csv> <out.md> [rep ...]"""
import collections, csv, json, os, subprocess, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]; ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        name = r[ki].split("(")[0].replace("void ", "").strip()
        agg[name].append(v)
    return agg

def rep_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
    allres = []
    for v in rows[2:]:
        res = {}
        for k in want:
            for i, name in enumerate(h):
                if name == k and i < len(v):
                    res[k] = (v[i], u[i])
        allres.append(res)
    return allres

def main():
    lc, outmd = sys.argv[1], sys.argv[2]
    reps = sys.argv[3:]
    agg = launches(lc)
    tot = sum(sum(x) for x in agg.values())
    lines = ["| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, x in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(x)} | {sum(x)/1e3:.2f} | {sum(x)/tot*100:.1f}% | {sum(x)/len(x):.1f} |")
    lines.append("")
    traffic = {}
    for rep in reps:
        for m in rep_metrics(rep):
            name = m.get("Kernel Name", ("?", ""))[0].split("(")[0].replace("void ", "").strip()
            lines.append(f"### {os.path.basename(rep)}: {name}")
            for k, (val, unit) in m.items():
                lines.append(f"- {k}: {val} {unit}")
            def tobytes(x):
                val, unit = x
                f = float(val.replace(",", ""))
                return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            if "dram__bytes_read.sum" in m and "launch__grid_size" in m:
                tb = tobytes(m["dram__bytes_read.sum"]) + tobytes(m["dram__bytes_write.sum"])
                base = name.split("<")[0].split("::")[-1]
                traffic[base] = {"bytes_per_launch": tb, "source": os.path.basename(rep)}
            lines.append("")
    if traffic:
        lines.append("traffic (dram read + write per captured launch): " + json.dumps(traffic))
    open(outmd, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

if __name__ == "__main__":
    main()

"""Summarise an ncu report's source page: top source lines by warp-stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
import os
kf = os.environ.get("NCU_KERNEL")
out = subprocess.run(["ncu", "-i", rep] + (["--kernel-name", "regex:" + kf] if kf else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]; idx = {h: i for i, h in enumerate(hdr)}
S = idx["Warp Stall Sampling (All Samples)"]
keys = [k for k in hdr if k.startswith("stall_") and "(Not" not in k]
data = []
for r in rows[3:]:
    if len(r) < len(hdr) or not r[0].isdigit(): continue
    try: s = int(r[S])
    except: continue
    data.append((s, int(r[0]), r[1].strip()[:70], {k[6:]: int(r[idx[k]]) for k in keys if r[idx[k]] not in ("", "0")}))
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for s, ln, src, st in sorted(data, reverse=True)[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s/tot*100:5.1f}% L{ln}: {src} | " + " ".join(f"{k}={v}" for k, v in top3))

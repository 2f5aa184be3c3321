"""Per-source-line executed instructions + stall samples of an ncu report (cuda,sass page)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]; idx = {}
for i, h in enumerate(hdr):
    idx.setdefault(h, i)
IE = idx["Instructions Executed"]; S = idx["Warp Stall Sampling (All Samples)"]
data = []
for r in rows[3:]:
    if len(r) < len(hdr) or not r[0].isdigit():
        continue
    try:
        n = int(r[IE] or 0); s = int(r[S] or 0)
    except ValueError:
        continue
    data.append((n, s, int(r[0]), r[1].strip()[:80]))
ti = sum(d[0] for d in data) or 1; ts = sum(d[1] for d in data) or 1
print(f"total warp-instructions {ti}, samples {ts}")
for n, s, ln, src in sorted(data, reverse=True)[:top]:
    print(f"inst {n/ti*100:5.1f}% samp {s/ts*100:5.1f}% L{ln}: {src}")

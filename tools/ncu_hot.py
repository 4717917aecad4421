"""Top stall lines of an ncu report's source page: python tools/ncu_hot.py rep [sass|cuda] [N]."""
import csv, subprocess, sys
rep = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "sass"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
args = ["ncu", "-i", rep, "--page", "source", "--csv"]
if mode == "cuda":
    args += ["--print-source", "cuda"]
out = subprocess.run(args, capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
i = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
data = [r for r in rows[1:] if len(r) == len(h)]
tot = sum(float(r[i] or 0) for r in data) or 1
print("total samples", tot)
for r in sorted(data, key=lambda r: -float(r[i] or 0))[:n]:
    print(f"{100*float(r[i] or 0)/tot:5.1f}%  {r[0][-5:]}  {r[src].strip()[:120]}")

"""Top SASS instructions by warp-stall samples for one kernel of an ncu report
(first launch of that kernel in the report)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--launch-count", "1"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r][0]
h = rows[hi]
si, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for i, r in enumerate(rows[hi + 1:]):
    if len(r) <= ai or not r[ai].strip().isdigit():
        break
    data.append((int(r[ai]), i, r[si].strip()))
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}")
for s, i, src in sorted(data, reverse=True)[:n]:
    print(f"{s:6d} {100*s/tot:5.1f}%  #{i:5d}  {src}")

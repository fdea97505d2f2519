"""Top SASS instructions of one kernel by warp-stall samples (ncu source page)."""
import csv
import io
import subprocess
import sys

path, regex = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{regex}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si = hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
ai = hdr.index("Address") if "Address" in hdr else 0
items = []
tot = 0
for r in rows[2:]:
    if len(r) < len(hdr) - 2:
        continue
    try:
        w = float(r[wi] or 0)
    except ValueError:
        continue
    tot += w
    items.append((w, r[ai], r[si]))
items.sort(reverse=True)
print(f"total stall samples {tot:.0f}")
for w, a, src in items[:top]:
    print(f"{100 * w / tot:5.1f}%  {a}  {src[:90]}")

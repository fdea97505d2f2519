"""Instruction histogram of one kernel from an ncu report (source page, SASS)."""
import csv
import io
import subprocess
import sys
from collections import Counter

path, regex = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{regex}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci, si = hdr.index("Instructions Executed"), hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
cnt, st, tot = Counter(), Counter(), 0
for r in rows[2:]:
    if len(r) < len(hdr) - 2:
        continue
    try:
        n = float(r[ci] or 0)
    except ValueError:
        continue
    toks = r[si].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    cnt[op] += n
    tot += n
    try:
        st[op] += float(r[wi] or 0)
    except ValueError:
        pass
print(f"total warp-instructions {tot:.4g}")
for k, v in cnt.most_common(24):
    print(f"{k:10s} {v / tot * 100:5.1f}%   stall samples {st[k]:.0f}")

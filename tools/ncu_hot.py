"""Top SASS lines of an ncu source-page CSV by stall samples and by
instructions executed (for reading a profile summarised on the GPU box)."""

import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
if len(rows) < 3:
    sys.exit("no source page")
h = rows[1]
ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss]) if r[iss].isdigit() else 0, int(r[ia]) if r[ia].isdigit() else 0, i, r[isrc]) for i, r in
        enumerate(rows[2:]) if len(r) > max(ia, iss)]
tot_s = sum(d[0] for d in data) or 1
tot_i = sum(d[1] for d in data) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
print("-- top 40 by stall samples")
for s, n, i, src in sorted(data, reverse=True)[:40]:
    print(f"{s / tot_s:6.3f} {n / tot_i:6.3f} {i:5d} {src[:90]}")
print("-- top 60 by instructions executed")
for s, n, i, src in sorted(data, key=lambda d: -d[1])[:60]:
    print(f"{s / tot_s:6.3f} {n / tot_i:6.3f} {i:5d} {src[:90]}")
if len(sys.argv) > 2:  # full listing of executed lines: index, warp instructions, stall samples, SASS
    with open(sys.argv[2], "w") as fh:
        for s, n, i, src in data:
            if n or s:
                fh.write(f"{i}\t{n}\t{s}\t{src[:100]}\n")

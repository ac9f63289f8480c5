"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        print("==", rows[i][1][:140])
        hdr = rows[i + 1]
        ci, si = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
        body = []
        j = i + 2
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            try:
                body.append((float(rows[j][ci] or 0), j - i - 2, rows[j][si]))
            except (ValueError, IndexError):
                pass
            j += 1
        tot = sum(v for v, _, _ in body) or 1
        for v, k, s in sorted(body, key=lambda t: -t[0])[:n]:
            print(f"{v / tot * 100:5.1f}% [{k:4d}] {s[:100]}")
        i = j
    else:
        i += 1

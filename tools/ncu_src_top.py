"""Top CUDA source lines by warp-stall samples from an `ncu --page source --csv --print-source cuda,sass`
export (tools/ncu_deep.sh): usage python tools/ncu_src_top.py file.csv [N]"""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname, func, hdr, out = "?", "?", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    st = {hdr[i]: f(r[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not" not in hdr[i]}
    out.append((f(r[4]), fname, r[0], r[1].strip()[:80], sorted(st.items(), key=lambda x: -x[1])[:3]))
tot = sum(o[0] for o in out)
print(func[:150])
print("total samples", tot)
for s, fn, ln, src, st in sorted(out, key=lambda o: -o[0])[:N]:
    print(f"{100 * s / tot:5.1f}% {fn}:{ln:>4} {src:80s} {[(k[6:], int(v)) for k, v in st if v]}")

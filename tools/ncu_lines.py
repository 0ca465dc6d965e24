"""Aggregate ncu source-page stall samples by CUDA source line.

  python tools/ncu_lines.py <rep.ncu-rep> [top] [line_lo line_hi]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 10 ** 9
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
fname = None
out = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) <= wi or r[0] == "":
        continue
    try:
        w = float(r[wi])
        ins = float(r[ii])
        ln = int(r[0])
    except ValueError:
        continue
    if not (lo <= ln <= hi):
        continue
    st = sorted(((float(r[i]) if r[i] not in ("", "-") else 0.0, h[6:]) for i, h in stall), reverse=True)[:3]
    out.append((w, ins, f"{fname}:{r[0]}", r[1][:70], st))
tot = sum(o[0] for o in out) or 1
print(f"total samples {tot:.0f}")
for w, ins, loc, src, st in sorted(out, reverse=True)[:top]:
    s = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
    print(f"{100 * w / tot:5.1f}% inst {ins:8.0f} {loc:16s} {src:70s} [{s}]")

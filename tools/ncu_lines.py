"""Per-CUDA-source-line instruction and stall-sample shares of one kernel from an ncu report
(`ncu -i REP --page source --csv --print-source cuda,sass`): python tools/ncu_lines.py REP KERNEL_REGEX"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hh = [i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"]][0]
h = rows[hh]
hi = hh - 2
ii, wi = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
lines, cur, fname = {}, None, "?"
for r in rows[hi + 1:]:
    if len(r) <= ii:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if not r[0].isdigit() and r[0]:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:100])
        continue
    x = lines.setdefault(cur, [0.0, 0.0])

    def num(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    x[0] += num(r[ii])
    x[1] += num(r[wi])
ti = sum(v[0] for v in lines.values()) or 1
tw = sum(v[1] for v in lines.values()) or 1
print(f"total warp instructions {ti:.3e}, stall samples {tw:.0f}")
for (fn, ln, src), (i, w) in sorted(lines.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if i / ti >= thr or w / tw >= thr:
        print(f"{fn[:12]:12s}{ln:5d} inst {i / ti:6.3f} stall {w / tw:6.3f}  {src}")

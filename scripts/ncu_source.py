"""Per-CUDA-source-line instruction counts and stall samples of the kernels in an ncu report
(needs -lineinfo):  python scripts/ncu_source.py rep.ncu-rep [function-substring] [top-N]"""
import csv
import io
import subprocess
import sys

rep, sub, top = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else ""), int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
func, path, data = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No" or func is None or sub not in func:
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            ie, ss = int(r[7] or 0), int(r[4] or 0)
        except ValueError:
            continue
        if ie or ss:
            data.setdefault(func, []).append((ie, ss, f"{path}:{r[0]}", r[1].strip()[:90]))
for f, d in data.items():
    ti = sum(x[0] for x in d) or 1
    ts = sum(x[1] for x in d) or 1
    print(f"== {f[:110]}\n   warp-inst {ti:.3e}  stall samples {ts}")
    for x in sorted(d, key=lambda x: -x[0])[:top]:
        print(f"{100*x[0]/ti:5.1f}% inst {100*x[1]/ts:5.1f}% stall  {x[2]:>12} {x[3]}")

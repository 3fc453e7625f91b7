"""Top CUDA source lines of one kernel in an ncu report, by PC samples
(ncu --page source --print-source cuda,sass; needs -lineinfo + --import-source).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
fname, rows, tot_s, tot_i = None, [], 0, 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Kernel Name") or r[0] == "":
        continue
    try:
        s, n = int(r[6]), int(r[7])
    except (ValueError, IndexError):
        continue
    tot_s += s
    tot_i += n
    rows.append((s, n, f"{fname}:{r[0]}", r[1].strip()[:90]))
rows.sort(key=lambda t: -t[0])
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, n, loc, src in rows[:top]:
    print(f"{100.0 * s / max(tot_s, 1):5.1f}% {100.0 * n / max(tot_i, 1):5.1f}%i  {loc:28s} {src}")

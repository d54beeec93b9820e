"""Per-source-line warp-stall attribution of one kernel in an ncu report (needs -lineinfo and
--import-source on).  Usage: python profiles/ncu_lines.py <report> <kernel regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name-base", "demangled", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    try:
        samp = int(r[4] or 0)
        ins = int(r[7] or 0)
    except ValueError:
        continue
    if samp == 0:
        continue
    st = {hdr[i][6:]: int(float(r[i] or 0)) for i in range(len(hdr))
          if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
    st = sorted(((k, v) for k, v in st.items() if v), key=lambda x: -x[1])[:3]
    rows.append((samp, ins, f"{fname}:{r[0]}", r[1].strip()[:60], st))
tot = sum(x[0] for x in rows) or 1
print(f"total samples {tot}")
for s, ins, loc, src, st in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100.0 * s / tot:5.1f}% {ins:>10d}  {loc:20s} {src:60s} {st}")

"""Per-source-line warp-stall samples of one kernel launch from an ncu report (-lineinfo builds).
Usage: python tools/ncu_hotlines.py report.ncu-rep kernel_regex [top] [launch_skip]"""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
col = 7 if (len(sys.argv) > 5 and sys.argv[5] == "inst") else 4  # 7: warp instructions executed
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--kernel-name", f"regex:{pat}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
res = []
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0].isdigit():
        try:
            res.append((int(float(r[col] or 0)), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
res.sort(reverse=True)
for s, loc, src in res[:top]:
    print(f"{100 * s / tot:5.1f}%  {loc:24s} {src}")

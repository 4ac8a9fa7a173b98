"""Per-source-line executed instructions and stall samples of an ncu report (dev tool).
usage: python tools/ncu_lines2.py report.ncu-rep [N] [cells]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cells = float(sys.argv[3]) if len(sys.argv) > 3 else 1.342e8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; cur = None; res = []
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if not r or hdr is None or not r[0].isdigit(): continue
    ie = r[hdr.index("Instructions Executed")]; sm = r[hdr.index("Warp Stall Sampling (All Samples)")]
    try:
        res.append((cur, int(r[0]), int(ie) if ie not in ("", "-") else 0, int(sm) if sm not in ("", "-") else 0, r[1][:95]))
    except ValueError:
        pass
ti = sum(x[2] for x in res) or 1; ts = sum(x[3] for x in res) or 1
print(f"total inst {ti} ({ti / cells:.2f}/cell)  samples {ts}")
for x in sorted(res, key=lambda x: -x[2])[:N]:
    print(f"{x[0][:12]:12s}:{x[1]:4d} {100 * x[2] / ti:5.1f}% {x[2] / cells:5.2f}/c stall {100 * x[3] / ts:5.1f}%  {x[4]}")

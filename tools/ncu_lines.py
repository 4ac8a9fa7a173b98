"""Top source lines of an ncu report by executed instructions and stall samples (dev tool).
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; cur = None; res = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not r or hdr is None:
        continue
    try:
        ie = r[hdr.index("Instructions Executed")]
        if not r[0].isdigit():
            continue
        sm = r[hdr.index("Warp Stall Sampling (All Samples)")]
        res.append((cur, int(r[0]), int(ie) if ie not in ("", "-") else 0, int(sm) if sm not in ("", "-") else 0, r[1][:90]))
    except Exception:
        pass
ti = sum(x[2] for x in res) or 1; ts = sum(x[3] for x in res) or 1
print(f"total inst {ti}  samples {ts}")
for x in sorted(res, key=lambda x: -x[3])[:N]:
    print(f"{x[0][:14]:14s}:{x[1]:4d} inst {100*x[2]/ti:5.1f}% stall {100*x[3]/ts:5.1f}%  {x[4]}")

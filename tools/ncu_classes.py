"""Group SASS instructions of an ncu report by execution count (= how often the code runs:
per window, per warp-step, per launch...) to find where the instruction budget goes (dev tool).
usage: python tools/ncu_classes.py report.ncu-rep [show_count]"""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
ins = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "Kernel Name":
        continue
    d = dict(zip(hdr, r))
    try:
        ie = int(d["Instructions Executed"])
    except Exception:
        continue
    ins.append((d["Source"].strip(), ie, int(d["Warp Stall Sampling (All Samples)"] or 0)))
tot = sum(i for _, i, _ in ins)
stall = sum(s for _, _, s in ins) or 1
by = collections.defaultdict(lambda: [0, 0, 0])
for s_, ie, st in ins:
    b = by[ie]
    b[0] += 1; b[1] += ie; b[2] += st
print(f"total executed {tot}")
for ie, (n, e, st) in sorted(by.items(), key=lambda x: -x[1][1])[:12]:
    print(f"exec-count {ie:>10d}: {n:5d} static instr, {100 * e / tot:5.1f}% of executed, {100 * st / stall:5.1f}% of stall samples")
if len(sys.argv) > 2:
    want = int(sys.argv[2])
    ops = collections.Counter(s.split()[1] if s.startswith("@") else s.split()[0] for s, ie, _ in ins if ie == want)
    print(ops.most_common(40))

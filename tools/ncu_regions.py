"""Aggregate an ncu source page (cuda,sass CSV) by kernel region (development tool).
usage: python tools/ncu_regions.py report.ncu-rep"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
hdr = None
cur = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] in ("", "Function Name") or hdr is None:
        continue
    try:
        ie = r[hdr.index("Instructions Executed")]
        res.append((cur, int(r[0]), int(ie) if ie not in ("", "-") else 0, int(r[4])))
    except Exception:
        pass
root = "/root/repo/paper_2211_00705_b200/csrc/"
marks = {}
for fname in ("eis_resident.cuh", "eis_device.cuh"):
    src = open(root + fname).read().split("\n")
    ms = []
    for i, l in enumerate(src, 1):
        m = re.search(r"-{6,} (S1|S2|P1|S4|S5|P2|remesh|creations|write back)", l)
        if m:
            ms.append((i, m.group(1)))
        m2 = re.match(r"__device__.*?\b(\w+)\(", l)
        if m2 and fname == "eis_device.cuh":
            ms.append((i, "dev:" + m2.group(1)))
        m3 = re.match(r"(?:template.*)?__device__.*?\b(dts_block|build_boundary_list|remesh_shift|edge_view|cell_update|region_at|tiny_at)\(", l)
        if m3 and fname == "eis_resident.cuh":
            ms.append((i, "fn:" + m3.group(1)))
        if "resident_steps(" in l and fname == "eis_resident.cuh":
            ms.append((i, "kernel-entry"))
    marks[fname] = sorted(ms)


def region(f, l):
    if f not in marks:
        return f
    name = "top"
    for i, nm in marks[f]:
        if l >= i:
            name = nm
    return name


agg = {}
for f, l, ie, smp in res:
    k = region(f, l)
    a = agg.setdefault(k, [0, 0])
    a[0] += ie
    a[1] += smp
tot = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{k:34s} inst {v[0]:12d} {100 * v[0] / tot:5.1f}%  stall-samples {100 * v[1] / ts:5.1f}%")

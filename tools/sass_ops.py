"""Opcode histogram of one kernel's SASS (development tool).
usage: python tools/sass_ops.py lib.so name-substring [N]"""
import collections, re, subprocess, sys
so, key = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
for sec in re.split(r"\n\s+Function : ", txt)[1:]:
    name = sec.split("\n", 1)[0].strip()
    if key not in name:
        continue
    ops = collections.Counter(re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", sec))
    print(name[:90], "total", sum(ops.values()))
    print("  ", ", ".join(f"{k} {v}" for k, v in ops.most_common(N)))

"""Per-kernel SASS instruction summary of libcascade.so (cuobjdump -sass):
counts of the opcodes that show which hardware path each kernel uses
(tcgen05 MMA = UTCHMMA/UTCQMMA, TMEM loads = LDTM, TMA/bulk copies =
UTMALDG/UBLKCP, mma.sync = HMMA, 128-bit global loads, barriers, spills).
usage: python scripts/sass_summary.py [lib.so] > profiles/<round>/sass_summary.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2506_20675_b200/libcascade.so"
WATCH = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "UBLKPF", "HMMA", "LDG.E.128", "LDG.E.NA.128",
         "LDG.E.64", "STG.E.128", "LDS", "STS", "ATOMG", "RED", "MEMBAR", "BAR.SYNC", "SYNCS", "STL", "LDL", "FENCE"]

txt = subprocess.check_output(["cuobjdump", "-sass", LIB], text=True, stderr=subprocess.DEVNULL)
kern = None
counts = collections.OrderedDict()
for line in txt.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts.setdefault(kern, collections.Counter())
        continue
    if kern is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    c = counts[kern]
    c["_total"] += 1
    for w in WATCH:
        if op == w or op.startswith(w + "."):
            c[w] += 1
            break


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out)) if len(out) == len(names) else {n: n for n in names}


dm = demangle(list(counts))
print(f"# SASS opcode summary of {LIB} (cuobjdump -sass; sm_100a)")
print("# kernel | total instructions | " + " ".join(WATCH))
for k, c in counts.items():
    name = re.sub(r"\(.*", "", dm[k]).replace("void ", "").replace("cascade::", "")
    tmpl = re.search(r"<.*>", dm[k])
    label = name if name.endswith(">") or not tmpl else name
    fields = " ".join(f"{w}={c[w]}" for w in WATCH if c[w])
    print(f"{label:60s} total={c['_total']:6d}  {fields}")

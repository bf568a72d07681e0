"""SASS instruction census of the built library: per kernel, the counts of the
Blackwell-specific mnemonics that show the tcgen05 / TMEM / TMA / bulk-copy
paths (UTCHMMA/UTCQMMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st, UTCBAR =
tcgen05.commit, UBLKCP / UBLKPF = cp.async.bulk / its L2 prefetch, UTMALDG =
tensor-map TMA, SYNCS = mbarrier ops), plus the total instruction count.
Usage: python scripts/sass_census.py [lib.so] > profiles/<round>/sass_census.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2504_21627_b200", "liblsnif_gpu.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "UBLKCP", "UBLKPF", "UTMALDG",
        "SYNCS", "HMMA", "FFMA", "LDS", "LDG", "STG", "SHFL", "ATOMG", "RED"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and kern:
        counts[kern]["_total"] += 1
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k):
                counts[kern][k] += 1
                break
demangled = {}
names = list(counts)
try:
    dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    demangled = dict(zip(names, dm))
except OSError:
    pass
print(f"# SASS census of {os.path.relpath(lib, ROOT)} (cuobjdump -sass, sm_100a)")
tot = collections.Counter()
for k, c in counts.items():
    tot.update(c)
    name = demangled.get(k, k)
    name = re.sub(r"\(.*", "", name.replace("(anonymous namespace)", "anon"))[:110]
    fields = " ".join(f"{key}={c[key]}" for key in KEYS if c[key])
    print(f"{name}: total={c['_total']} {fields}")
print("ALL: " + " ".join(f"{key}={tot[key]}" for key in ["_total"] + KEYS if tot[key]))

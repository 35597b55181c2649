"""SASS opcode histogram per kernel of libxlmimo_b200.so (cuobjdump -sass):
the instructions that prove tcgen05 / TMA / DMMA use.
    python tools/sass_hist.py [lib.so] > profiles/r02_sass_hist.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2305_13925_b200/_native/libxlmimo_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
WATCH = ["UTCHMMA", "UTCHMMA.2CTA", "UTCQMMA", "UTCBAR", "UTCBAR.2CTA", "UTCCP", "UTCATOMSWS", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UTMASTG",
         "UTMAPF", "SYNCS", "ELECT", "HMMA", "DMMA", "DFMA", "FFMA", "FMUL", "F2FP", "LDS", "STS", "LDG", "STG", "SHFL"]
funcs = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        funcs[cur][m.group(1)] += 1
        if m.group(2) and ".2CTA" in m.group(2):  # cta_group::2 (CTA-pair) forms, counted also on their own
            funcs[cur][m.group(1) + ".2CTA"] += 1


def short(name):
    try:
        d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        d = name
    return re.sub(r"\(.*", "", d)[:60]


print("| kernel | " + " | ".join(WATCH) + " | total |")
print("|---|" + "---|" * (len(WATCH) + 1))
for f, c in funcs.items():
    if sum(c[w] for w in WATCH[:12]) == 0 and "DMMA" not in c:
        continue
    print(f"| `{short(f)}` | " + " | ".join(str(c[w]) for w in WATCH) + f" | {sum(c.values())} |")

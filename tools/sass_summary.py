"""Instruction summary of the product kernels from `cuobjdump -sass libellm.so`: per kernel, the
counts of the SASS mnemonics that show which hardware paths it uses (TMA, bulk copies, tcgen05
MMA / TMEM, HMMA, mbarrier sync, MUFU) and its register / shared-memory use from -res-usage.
Usage: python tools/sass_summary.py > profiles/r02_sass.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2506_15155_b200", "libellm.so")
KEYS = ["UTMALDG", "UTMASTG", "UBLKCP", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS",
        "HMMA", "SYNCS", "MUFU.EX2", "LDS", "STS", "LDG", "STG", "ATOMG", "REDG", "MEMBAR", "FENCE"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    funcs[cur][k] += 1
    usage = {}
    for line in res.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
        if m and cur:
            usage[cur] = (int(m.group(1)), int(m.group(2)))
    names = demangle(list(funcs))
    print("| kernel | regs | static smem | " + " | ".join(KEYS) + " |")
    print("|---|---|---|" + "---|" * len(KEYS))
    for f, c in funcs.items():
        r, sm = usage.get(f, ("?", "?"))
        short = names[f].replace("(anonymous namespace)::", "").replace("void ", "")
        short = re.sub(r"\(.*", "", short)
        print(f"| `{short}` | {r} | {sm} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")


if __name__ == "__main__":
    sys.exit(main())

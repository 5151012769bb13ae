"""Per-kernel SASS instruction census of the built libraries (development aid):
proves which hardware paths each kernel uses (UTMALDG = TMA tensor load, UTMAPF =
TMA L2 prefetch, UTMASTG = TMA tensor store, HMMA = mma.sync, UTCHMMA/UTCBAR =
tcgen05.mma / commit, LDTM / STTM = tcgen05.ld / st, MUFU = ex2, ...).

  python tools/sass_census.py [lib.so ...] > profiles/rNN_sass_census.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = ["UTMALDG", "UTMAPF", "UTMASTG", "UBLKCP", "HMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "MUFU", "FFMA2",
       "FADD2", "FMUL2", "FMNMX3", "FMNMX", "FFMA", "PRMT", "LOP3", "SHFL", "LDS", "STS", "LDG", "STG", "RED",
       "ATOM", "ATOMG", "MEMBAR", "SYNCS", "BAR", "ELECT"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
        return out[:len(names)]
    except Exception:
        return names


def census(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
        if cur and m:
            op = m.group(1)
            full = op + (m.group(2) or "")
            kernels[cur][op] += 1
            if op == "FFMA" and ".F32x2" in full.upper():
                kernels[cur]["FFMA2"] += 1
    return kernels


def main():
    libs = sys.argv[1:] or [os.path.join(ROOT, "paper_2411_01142_b200", "libneo.so")]
    print("# SASS instruction census (`cuobjdump -sass`, static counts per kernel)\n")
    print("Static instruction counts in each kernel's SASS (not executed counts).  UTMALDG = TMA tensor load, "
          "UTMAPF = TMA L2 prefetch, UTMASTG = TMA store, HMMA = mma.sync, UTCHMMA = tcgen05.mma, "
          "UTCBAR = tcgen05.commit, LDTM / STTM = tcgen05.ld / st.\n")
    for lib in libs:
        ks = census(lib)
        names = demangle(list(ks))
        cols = [k for k in KEY if any(c.get(k) for c in ks.values())]
        print(f"## `{os.path.relpath(lib, ROOT)}`\n")
        print("| kernel | total | " + " | ".join(cols) + " |")
        print("|---|---|" + "---|" * len(cols))
        for (raw, c), nm in zip(ks.items(), names):
            short = re.sub(r"\(CUtensorMap_st.*|\(neo::.*", "", nm).replace("neo::(anonymous namespace)::", "")
            print(f"| `{short}` | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) for k in cols) + " |")
        print()


if __name__ == "__main__":
    main()

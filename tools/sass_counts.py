"""Per-kernel counts of the SASS instructions that prove which hardware path
each kernel uses (tcgen05 MMA / TMEM / TMA / bulk copies / DMMA), from
cuobjdump -sass of the shipped library:

    python tools/sass_counts.py [lib.so] > profiles/r02_sass_counts.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_11953_b200/libmpsvd_b200.so"
KEYS = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "DMMA",
        "HMMA", "IMMA", "LDGSTS", "SYNCS", "DFMA", "DADD", "DMUL", "MUFU"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    counts[cur][k] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    print(f"# SASS instruction counts per kernel, cuobjdump -sass {LIB} (sm_100a)")
    print("# " + " ".join(KEYS))
    for (name, c), d in zip(counts.items(), dem):
        short = re.sub(r"\(.*", "", d)
        cells = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
        print(f"{short}: {cells}")


if __name__ == "__main__":
    main()

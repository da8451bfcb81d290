"""Per-kernel SASS instruction counts of libosph.so (static, from cuobjdump -sass).

    python tools/sass_counts.py [paper_1403_4661_b200/libosph.so] > profiles/sass_r02.txt

Evidence that each kernel runs on the units DESIGN.md says it does:
DMMA.8x8x4 (fp64 tensor core MMA), DFMA (fp64 FMA pipe), UBLKCP (bulk
async copy = the TMA engine's cp.async.bulk), LDGSTS (cp.async 16-byte
global->shared), SYNCS (mbarrier arrive / wait / transaction counts), REDG
(global reductions), BAR (CTA barriers) and UCGABAR (cluster barriers).
"""

import re
import subprocess
import sys
from collections import Counter, defaultdict

OPS = ["DMMA.8x8x4", "DFMA", "DADD", "DMUL", "UBLKCP", "LDGSTS", "SYNCS", "REDG", "ATOMS", "BAR.SYNC",
       "UCGABAR", "MEMBAR", "FENCE"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1403_4661_b200/libosph.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    counts = defaultdict(Counter)
    func = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            func = m.group(1)
            continue
        if func is None or "/*" not in line:
            continue
        body = line.split("*/", 1)[-1] if line.strip().startswith("/*") else line
        for op in OPS:
            if re.search(r"\b" + re.escape(op), body):
                counts[func][op] += 1
    demangled = {}
    try:
        out = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
        demangled = dict(zip(counts, out))
    except OSError:
        pass
    print(f"# static SASS instruction counts per kernel: cuobjdump -sass {lib}")
    print("# (instructions in the binary, not executions)")
    print(f"{'kernel':60s} " + " ".join(f"{op:>10s}" for op in OPS))
    for func in sorted(counts, key=lambda f: demangled.get(f, f)):
        name = demangled.get(func, func)
        name = re.sub(r"\(.*", "", name)[:60]
        print(f"{name:60s} " + " ".join(f"{counts[func][op]:>10d}" for op in OPS))


if __name__ == "__main__":
    main()

"""Reference CSV reports for the GPU experiment harness.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_experiments.py

Runs the REFERENCE's own CLI (optisph.cli.main, pkg/src/optisph/cli.py:244-253)
from /root/reference/pkg/src on small band limits and writes its reports to
tests/golden/experiments/: exp1/exp2 accuracy sweeps, an error surface and a
conditioning profile.  tests/test_gpu_experiments.py runs the same commands
through paper_1403_4661_b200.cli on the GPU and compares row by row.
"""

import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

OUT = Path(__file__).resolve().parent / "experiments"

COMMANDS = {
    "exp1.csv": ["exp1", "-L", "8,16,32", "--trials", "3", "--seed", "5"],
    "exp2.csv": ["exp2", "-L", "8,16,32", "--trials", "3", "--seed", "6"],
    "errsurface.csv": ["errsurface", "-L", "16", "--trials", "2", "--seed", "7"],
    "cond_interleaved.csv": ["cond", "-L", "16,32"],
    "cond_condmin.csv": ["cond", "-L", "16,32", "--ordering", "condmin"],
}


def main():
    from optisph.cli import main as ref_main

    OUT.mkdir(parents=True, exist_ok=True)
    for name, argv in COMMANDS.items():
        rc = ref_main(argv + ["-o", str(OUT / name)])
        print(name, "rc", rc)


if __name__ == "__main__":
    main()

"""A/B timing of library builds with the same C-ABI: alternate runs of
tools/one_solve.py --time under HFB_LIBRARY=<lib>, report the median per lib.

    python tools/ab.py --rounds 3 A.so B.so [-- one_solve args]
"""
import os
import re
import statistics
import subprocess
import sys

args = sys.argv[1:]
rounds = 3
if args and args[0] == "--rounds":
    rounds, args = int(args[1]), args[2:]
extra = []
if "--" in args:
    i = args.index("--")
    args, extra = args[:i], args[i + 1:]
here = os.path.dirname(os.path.abspath(__file__))
times = {lib: [] for lib in args}
for _ in range(rounds):
    for lib in args:
        env = dict(os.environ, HFB_LIBRARY=os.path.abspath(lib))
        out = subprocess.run([sys.executable, os.path.join(here, "one_solve.py"), "--time",
                              "--reps", "5", *extra], env=env, capture_output=True,
                             text=True).stdout
        m = re.search(r"ms/solve=([0-9.]+)", out)
        times[lib].append(float(m.group(1)) if m else float("nan"))
for lib, ts in times.items():
    print(f"{lib}: median {statistics.median(ts):.3f} ms  {ts}")

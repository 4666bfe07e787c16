"""A/B kernel timing: run tools/kbench.py against several builds of libobg.so.

    python tools/ab.py --libs a.so,b.so --runs "model --scene c3" "build --scene uniform --levels 6"

Each (lib, run) pair is a fresh process (OBG_LIB_PATH selects the build);
rounds are interleaved so clock drift hits every variant alike; the best
time per pair is printed.
"""
import argparse
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--runs", nargs="+", required=True)
    a = ap.parse_args()
    libs = a.libs.split(",")
    best = {}
    digests = {}
    for _ in range(a.rounds):
        for run in a.runs:
            for lib in libs:
                env = dict(os.environ, OBG_LIB_PATH=os.path.abspath(lib))
                res = subprocess.run([sys.executable, os.path.join(REPO, "tools", "kbench.py")] + run.split(),
                                     capture_output=True, text=True, env=env, cwd=REPO)
                m = re.search(r": ([0-9.]+) us", res.stdout)
                if not m:
                    print(lib, run, "FAILED", res.stdout[-500:], res.stderr[-1500:], flush=True)
                    continue
                us = float(m.group(1))
                d = re.search(r"model=([0-9a-f]+)", res.stdout)
                if d:
                    digests.setdefault(run, {})[lib] = d.group(1)
                key = (run, lib)
                best[key] = min(best.get(key, 1e30), us)
    for run in a.runs:
        print(run)
        for lib in libs:
            print(f"   {lib:50s} {best.get((run, lib), float('nan')):9.1f} us  {digests.get(run, {}).get(lib, '')}")


if __name__ == "__main__":
    main()

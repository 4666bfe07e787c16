"""Run bench.py over every BASELINE.json shape and tabulate (GPU box).

    python tools/sweep.py OUT_PREFIX      -> OUT_PREFIX.jsonl, OUT_PREFIX.md
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = [("C0", ["--config", "0"]), ("C1", ["--config", "1"]), ("C2", ["--config", "2"]),
        ("C3 (headline)", ["--config", "3"])]
for v in ("uniform", "constant"):
    for L in (4, 5, 6, 7):
        RUNS.append((f"C4 {v} L{L}", ["--config", "4", "--levels", str(L), "--variant", v]))


def main():
    prefix = sys.argv[1]
    rows = []
    with open(prefix + ".jsonl", "w") as out:
        for name, extra in RUNS:
            cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--steps", "10", "--warmup", "3",
                   "--no-cpu-baseline", "--no-e2e"] + extra
            res = subprocess.run(cmd, capture_output=True, text=True, cwd=REPO)
            line = next((ln for ln in reversed(res.stdout.splitlines()) if ln.startswith("{")), None)
            if line is None:
                print(name, "FAILED", res.stderr[-2000:], file=sys.stderr)
                continue
            out.write(line + "\n")
            rows.append((name, json.loads(line)))
    with open(prefix + ".md", "w") as md:
        md.write("# Sweep: bench.py over every BASELINE.json shape (tools/sweep.py)\n\n")
        md.write("Each line parity-checks the timed outputs against the reference's recorded outputs.\n")
        md.write("frac = achieved / MEASURED_PEAKS.json hbm_gbs; classify 4 B/px, build 3 B/px (+ leaf cube).\n\n")
        md.write("| workload | step ms | value Mpx/s | build ms | classify ms | classify frac | build frac | parity |\n")
        md.write("|---|---|---|---|---|---|---|---|\n")
        for name, d in rows:
            c, ph = d["config"], d["phases"]
            par = d.get("parity") or {}
            ok = all(v for k, v in par.items() if k != "frames") if par else None
            md.write(f"| {name}: {c['workload'].split(':')[0]} | {d['ms_per_step']} | {d['value']:,.0f} | "
                     f"{ph['build_ms']} | {ph['classify_ms']} | {d['roofline']['frac']} | {ph['build_hbm_frac']} | "
                     f"{ok} |\n")


if __name__ == "__main__":
    main()

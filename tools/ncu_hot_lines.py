"""Top SASS lines of a kernel by warp-stall samples, from `ncu -i REP --page source --csv`.

    python tools/ncu_hot_lines.py source.csv [N] > profiles/<name>.md
"""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    name = rows[0][1] if rows and rows[0][0] == "Kernel Name" else "?"
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) >= len(hdr) - 2]
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    samples = lambda r: int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    total = sum(samples(r) for r in body)
    inst = sum(int(r[col["Instructions Executed"]] or 0) for r in body)
    print(f"# ncu source page: `{name[:70]}`\n")
    print(f"{len(body)} SASS lines, {inst:,} warp instructions, {total:,} stall samples.\n")
    agg = {h: sum(int(r[col[h]] or 0) for r in body) for h in stall_cols}
    print("Stall samples by reason: " + ", ".join(f"{h[6:]} {v * 100 // max(total, 1)} %" for h, v in
                                                  sorted(agg.items(), key=lambda kv: -kv[1])[:8]) + "\n")
    print("| # | SASS | samples | % | warp inst | top stall |")
    print("|---|---|---|---|---|---|")
    for k, r in enumerate(sorted(body, key=samples, reverse=True)[:top]):
        st = max(stall_cols, key=lambda h: int(r[col[h]] or 0))
        print(f"| {k + 1} | `{r[col['Source']].strip()[:60]}` | {samples(r)} | {samples(r) * 100 / max(total, 1):.1f} | "
              f"{r[col['Instructions Executed']]} | {st[6:]} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

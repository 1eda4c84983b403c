"""Per-kernel share of the last step in an ncu launch list (the
`--metrics gpu__time_duration.sum` CSV of `bench.py --quick`): the launches
after the last k_tc_prep_c (or, without one, the last len(step) launches).
usage: python tools/launch_shares.py launches.csv out.json"""
import csv
import json
import sys


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            rows.append((name.strip(), float(r["Metric Value"].replace(",", "")) / 1e3))
    starts = [i for i, (n, _) in enumerate(rows) if n.startswith("k_tc_prep_c")]
    first = starts[-1] if starts else max(0, len(rows) - 8)
    if first > 0 and rows[first - 1][0].startswith("k_zero_rows"):
        first -= 1  # the zero fill of the empty rows is launched (side stream) before the C split
    step = rows[first:]
    total = sum(us for _, us in step)
    out = {"source": sys.argv[1] + " (ncu --metrics gpu__time_duration.sum --clock-control none "
                     "-k regex:^k_ over `bench.py --quick --steps 2 --warmup 1`; the list also "
                     "holds the inspector and plan-creation kernels)",
           "last_step_launches": {}, "sum_ms": total / 1e3,
           "note": "serialised cold-cache launches: shares, not absolutes (the bench step "
                   "overlaps the zero fill with the first op and the long-row segments with the "
                   "short-row kernel)"}
    for n, us in step:
        e = out["last_step_launches"].setdefault(n, {"us": 0.0, "share": 0.0})
        e["us"] += us
        e["share"] = e["us"] / total
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

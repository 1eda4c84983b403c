"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
from an ncu report of `bench.py --quick` and record it for bench.py's
roofline.traffic field.

usage: python tools/traffic.py <report.ncu-rep> <config> <stage>...
  stages are matched to the captured launches in order (e.g. first_op wave1_spmm);
  "name:N" sums N consecutive launches into one stage, "-" skips a launch
writes/updates profiles/ncu_traffic.json: {config: {stage: {kernel, bytes, ...}}}
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * scale


def main():
    rep, cfg, stages = sys.argv[1], sys.argv[2], sys.argv[3:]
    rows = summarise(rep)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    d = data.setdefault(cfg, {})
    # a stage may span several launches: "wave1_spmm:3" sums the next three;
    # "-" skips a launch (e.g. a small prep kernel)
    k = 0
    for spec in stages:
        name, _, cnt = spec.partition(":")
        cnt = int(cnt or 1)
        group = rows[k:k + cnt]
        k += cnt
        if name == "-":
            continue
        rd = sum(to_bytes(r["dram__bytes_read.sum"], r.get("dram__bytes_read.sum.unit", "byte"))
                 for r in group)
        wr = sum(to_bytes(r["dram__bytes_write.sum"], r.get("dram__bytes_write.sum.unit", "byte"))
                 for r in group)
        tus = sum(float(r["gpu__time_duration.sum"]) * (1e3 if r.get("gpu__time_duration.sum.unit") == "ms" else 1.0)
                  for r in group)
        d[name] = {"kernel": " + ".join(r["kernel"][:60] for r in group), "dram_bytes": rd + wr,
                   "dram_read": rd, "dram_write": wr, "ncu_time_us": tus, "launches": cnt,
                   "source": os.path.basename(rep)}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()

"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
from an ncu report of `bench.py --quick` and record it for bench.py's
roofline.traffic field.

usage: python tools/traffic.py <report.ncu-rep> <config> <stage>...
  stages are matched to the captured launches in order (e.g. first_op wave1_spmm)
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
    for stage, r in zip(stages, rows):
        rd = to_bytes(r["dram__bytes_read.sum"], r.get("dram__bytes_read.sum.unit", "byte"))
        wr = to_bytes(r["dram__bytes_write.sum"], r.get("dram__bytes_write.sum.unit", "byte"))
        d[stage] = {"kernel": r["kernel"][:120], "dram_bytes": rd + wr, "dram_read": rd,
                    "dram_write": wr, "ncu_time_us": r["gpu__time_duration.sum"],
                    "source": os.path.basename(rep)}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()

"""Sweep SpMM kernel variants (TFG_SPMM_VARIANT) on a BASELINE config and
print per-stage device times.  Each variant runs in a fresh process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2407_00243_b200 as P
from paper_2407_00243_b200 import workloads as W
w = W.make(%r)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
plan = P.Plan(prob, P.build_schedule(prob.a, w.scheduler_config()))
out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device="cuda")
fl = torch.empty(64 << 20, device="cuda")
res = {}
for k in range(12):
    fl.fill_(k); r = plan.profile(out)
    if k >= 2:
        for name, ms, by in r: res.setdefault(name, []).append((ms, by))
print(json.dumps({k: [float(np.median([m for m, _ in v])), v[0][1] / float(np.median([m for m, _ in v])) / 1e6] for k, v in res.items()}))
'''


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["-1"] + [str(k) for k in range(11)]
    for spec in variants:
        env = dict(os.environ)
        # composite codes: "S1+D3" applies each part's environment in turn
        parts = spec.split("+")
        for extra in [q for q in parts if q.startswith("@")]:  # "@VAR=value": any env knob
            k_, v_ = extra[1:].split("=", 1)
            env[k_] = v_
        parts = [q for q in parts if not q.startswith("@")] or ["-1"]
        for extra in parts[:-1]:
            key = {"X": "TFG_BAND_DIA_EXEC", "D": "TFG_SWEEP_DBG", "S": "TFG_SWEEP",
                   "R": "TFG_TC_RING", "T": "TFG_TC_DBG"}.get(extra[:1])
            if key:
                env[key] = extra[1:]
        v = parts[-1]
        if v.startswith("X"):  # stencil (DIA-window) band consumer on/off at execution
            env["TFG_BAND_DIA_EXEC"] = v[1:]
            v = "-1"
        if v.startswith("D"):  # band sweep debug mask (timing only)
            env["TFG_SWEEP_DBG"] = v[1:]
            v = "-1"
        if v.startswith("S"):  # dependency-driven band sweep on/off
            env["TFG_SWEEP"] = v[1:]
            v = "-1"
        if v.startswith("R"):  # tensor-core raw ring depth
            env["TFG_TC_RING"] = v[1:]
            v = "-1"
        if v.startswith("T"):  # tensor-core kernel debug mask (timing only)
            env["TFG_TC_DBG"] = v[1:]
            v = "-1"
        if v.startswith("r"):  # ring-gather depth for skewed lists
            env["TFG_RING"] = v[1:]
            v = "-1"
        if v.startswith("G"):  # GEMM variant
            env["TFG_GEMM_VARIANT"] = v[1:]
            v = "-1"
        if v.startswith("u0"):  # band without the mini-group union consumer
            env["TFG_BAND_UNION"] = "0"
            v = v[2:] or "-1"
        if v.startswith("s"):  # skewed strip variant
            env["TFG_SKEW_VARIANT"] = v[1:]
            v = "-1"
        if v.startswith("v2"):
            env["TFG_BAND_V"] = "2"
            v = v[2:]
        if v.startswith("w"):  # w<stages>_<kb>: warp-specialised band kernel
            st_, kb = v[1:].split("_")
            env["TFG_BAND_WS"] = st_
            env["TFG_BAND_KB"] = kb
            v = "-1"
        if v.startswith("b"):
            env["TFG_BAND_KB"] = v[1:]
            env["TFG_BAND_WS"] = "0"
            v = "-1"
        if v.startswith("n"):
            env["TFG_SPMM_BAND"] = "0"
            v = "-1"
        if v.startswith("g"):
            env["TFG_SPMM_GROUPS"] = "1"
            v = v[1:] or "-1"
        v = int(v)
        if v >= 0:
            env["TFG_SPMM_VARIANT"] = str(v)
        r = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg)], capture_output=True, text=True, env=env)
        print(cfg, "variant", spec, r.stdout.strip() or r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()

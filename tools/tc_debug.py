"""Localise tensor-core first-op differences against the FFMA path (TFG_TC=0):
per row of D, report the error and whether the row is fused (wavefront 0) or
computed in wavefront 1.  usage: python tools/tc_debug.py [banded|cfg3]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402


def problem(kind):
    if kind == "banded":
        n, bc, cc, hb = 20000, 64, 64, 2
        rows = [np.arange(max(0, i - hb), min(n, i + hb + 1)) for i in range(n)]
        rp = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int32)
        ci = np.concatenate(rows).astype(np.int32)
        rng = np.random.default_rng(4)
        v = rng.uniform(-1, 1, ci.size)
        a = P.Csr(n, n, rp, ci, v)
        b = rng.standard_normal((n, bc)).astype(np.float32)
        c = (rng.standard_normal((bc, cc)) / 8).astype(np.float32)
        cfg = P.SchedulerConfig(ct_size=512, num_workers=3, cache_size_words=10 ** 9, b_cols=bc,
                                c_cols=cc, index_to_scalar_ratio=1.0)
        return a, b, c, cfg
    w = W.make(kind, scale=1 / 8 if kind == "cfg3" else 1 / 64)
    return w.a, w.b, w.c, w.scheduler_config()


def run(a, b, c, s, tc):
    os.environ["TFG_TC"] = "1" if tc else "0"
    prob = P.DeviceProblem(a, b, c, np.float32)
    return P.Plan(prob, s).execute().cpu().numpy()


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "banded"
    a, b, c, cfg = problem(kind)
    s = P.build_schedule(a, cfg)
    flat = s.export() if hasattr(s, "export") else None
    want = run(a, b, c, s, False)
    got = run(a, b, c, s, True)
    un_t = run(a, b, c, None, True)
    un_f = run(a, b, c, None, False)
    scale = np.abs(want).max()
    err = np.abs(got - want).max(axis=1) / scale
    print("fused tc vs ffma max", err.max(), "bad rows", int((err > 1e-5).sum()), "of", len(err))
    print("unfused tc vs ffma max", (np.abs(un_t - un_f).max() / scale))
    bad = np.nonzero(err > 1e-5)[0]
    print("first bad rows", bad[:20].tolist())
    if flat is not None:
        print(flat.keys() if isinstance(flat, dict) else type(flat))


if __name__ == "__main__":
    main()

"""Column popularity of a BASELINE config's A: share of the nonzeros that fall
in the K most-gathered columns (the best hit rate an L2 holding K rows of D1
could reach).  usage: python tools/col_popularity.py cfg5"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
w = W.make(name)
cnt = np.bincount(w.a.col_idx, minlength=w.n).astype(np.int64)
srt = np.sort(cnt)[::-1]
cum = np.cumsum(srt)
nnz = int(cum[-1])
row_bytes = w.c_cols * np.dtype(w.dtype).itemsize
out = {"config": name, "n": int(w.n), "nnz": nnz, "row_bytes": int(row_bytes), "top": {}}
for k in [256, 1024, 4096, 16384, 65536, 131072, 262144, 393216, 524288, 786432, 1048576, 2097152,
          4194304]:
    if k <= w.n:
        out["top"][str(k)] = {"mb": k * row_bytes / 2**20, "share": float(cum[k - 1] / nnz),
                              "min_count": int(srt[k - 1])}
rl = np.diff(w.a.row_ptr.astype(np.int64))
out["rows_empty"] = int((rl == 0).sum())
out["row_len_pct"] = {str(p): float(np.percentile(rl, p)) for p in (50, 90, 99, 99.9, 100)}
print(json.dumps(out, indent=1))

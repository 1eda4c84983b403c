"""Host-side mirror of the reference ``tilefuse`` operator API over libtfg.

The reference exposes the path as C++ templates (include/tilefuse/*.hpp) and
a pybind module ``tilefuse._core`` (python/bindings.cpp).  This module keeps
the names, argument meaning and error behaviour of both, with the compute on
the B200 through the C-ABI in include/tfg.h:

* ``SchedulerConfig``        -- scheduler.hpp:15-24
* ``Csr``                    -- csr.hpp:19-72 (validated like ``checked``)
* ``build_schedule``         -- scheduler.hpp:300-301 (GPU inspector)
* ``Schedule.fused_ratio``   -- scheduler.hpp:304
* ``validate_schedule``      -- scheduler.hpp:308-310
* ``schedule_to_json`` / ``schedule_from_json`` -- schedule_io.cpp:9-54
* ``fused_gemm_spmm`` / ``fused_spmm_spmm`` / ``unfused_*`` -- kernels.hpp:182-236
  (and the bindings' numpy-in / numpy-out lambdas, bindings.cpp:143-191)
* ``DeviceProblem`` + ``Plan`` -- "inspect once, execute many" with
  device-resident operands (no host<->device traffic per execution).

Errors: std::invalid_argument -> ValueError, std::runtime_error ->
RuntimeError, as pybind11 translates them for the reference module.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TFG_F32, TFG_F64, TfgConfig, TfgProblem, check, i32p, i64p, f64p, lib

DEFAULT_CACHE_WORDS = 160 * 1024


@dataclass
class SchedulerConfig:
    """tilefuse::SchedulerConfig with the reference defaults (scheduler.hpp:15-24)."""

    ct_size: int = 2048
    num_workers: int = 1
    cache_size_words: int = DEFAULT_CACHE_WORDS
    b_cols: int = 32
    c_cols: int = 32
    index_to_scalar_ratio: float = 0.5
    b_is_dense: bool = True
    whole_b_cost: bool = False

    def to_c(self) -> TfgConfig:
        return TfgConfig(int(self.ct_size), int(self.num_workers), int(self.cache_size_words),
                         int(self.b_cols), int(self.c_cols), float(self.index_to_scalar_ratio),
                         int(bool(self.b_is_dense)), int(bool(self.whole_b_cost)))


def _dt_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return TFG_F64
    if dt == np.float32:
        return TFG_F32
    raise ValueError(f"unsupported dtype {dt} (float32 or float64)")


# ---------------------------------------------------------------------------
# CSR (csr.hpp)
# ---------------------------------------------------------------------------
class Csr:
    """Host CSR matrix; validated on construction like CsrMatrix::checked
    (csr.hpp:36-71): row_ptr[0]=0, non-decreasing, columns strictly
    increasing per row and inside [0, n_cols)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values, dtype=None, validate=True):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        vals = np.asarray(values)
        if dtype is None:
            dtype = vals.dtype if vals.dtype in (np.float32, np.float64) else np.float64
        self.values = np.ascontiguousarray(vals, dtype=dtype)
        if validate:
            self.validate()

    def validate(self):
        if self.n_rows < 0 or self.n_cols < 0:
            raise ValueError("csr: negative dimension")
        if self.row_ptr.ndim != 1 or self.row_ptr.size != self.n_rows + 1:
            raise ValueError("csr: row_ptr length != n_rows + 1")
        if self.row_ptr[0] != 0:
            raise ValueError("csr: row_ptr[0] != 0")
        d = np.diff(self.row_ptr.astype(np.int64))
        if (d < 0).any():
            raise ValueError(f"csr: row_ptr not non-decreasing at row {int(np.argmax(d < 0))}")
        nz = int(self.row_ptr[-1])
        if self.col_idx.size != nz or self.values.size != nz:
            raise ValueError("csr: col_idx/values length != nnz")
        if nz:
            if (self.col_idx < 0).any() or (self.col_idx >= self.n_cols).any():
                bad = int(np.argmax((self.col_idx < 0) | (self.col_idx >= self.n_cols)))
                r = int(np.searchsorted(self.row_ptr, bad, side="right") - 1)
                raise ValueError(f"csr: column out of range in row {r}")
            inc = np.diff(self.col_idx.astype(np.int64)) > 0
            first = np.zeros(nz, bool)
            starts = self.row_ptr[:-1][d > 0]
            first[starts] = True
            ok = first[1:] | inc
            if not ok.all():
                bad = int(np.argmax(~ok)) + 1
                r = int(np.searchsorted(self.row_ptr, bad, side="right") - 1)
                raise ValueError(f"csr: columns not strictly increasing in row {r}")

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.row_ptr.size else 0

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def square(self) -> bool:
        return self.n_rows == self.n_cols

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols), np.float64)
        rows = np.repeat(np.arange(self.n_rows), self.row_nnz())
        out[rows, self.col_idx] = self.values
        return out

    def astype(self, dtype) -> "Csr":
        return Csr(self.n_rows, self.n_cols, self.row_ptr, self.col_idx,
                   self.values.astype(dtype), validate=False)

    def __repr__(self):
        return f"Csr({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


def gen_random_sparse(n: int, density: float, seed: int = 42) -> Csr:
    """generate.hpp:15-63 (bindings.cpp:111-112); host-side, see generate.py."""
    from .generate import gen_random_sparse as g

    return g(n, density, seed)


def gen_banded(n: int, half_bandwidth: int) -> Csr:
    """generate.hpp:66-94 (bindings.cpp:113-114); host-side, see generate.py."""
    from .generate import gen_banded as g

    return g(n, half_bandwidth)


def choose_tile_size(n: int, num_workers: int, ct_size: int) -> int:
    """scheduler.cpp:124-129."""
    out = C.c_int32()
    check(lib().tfg_choose_tile_size(int(n), int(num_workers), int(ct_size), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# Schedule (scheduler.hpp) -- device resident
# ---------------------------------------------------------------------------
class Schedule:
    """Device-resident FusedSchedule handle (tfg_schedule)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        n, t = C.c_int32(), C.c_int32()
        nt = (C.c_int64 * 2)()
        nj = (C.c_int64 * 2)()
        secs = C.c_double()
        check(lib().tfg_schedule_info(self._h, C.byref(n), C.byref(t), nt, nj, C.byref(secs)))
        self.n = n.value
        self.tile_size = t.value
        self.num_tiles_per_wave = (nt[0], nt[1])
        self.num_jrows_per_wave = (nj[0], nj[1])
        self.inspect_seconds = secs.value
        self._flat = None

    @property
    def handle(self):
        return self._h

    def num_tiles(self) -> int:
        return int(sum(self.num_tiles_per_wave))

    def fused_ratio(self) -> float:
        return float(lib().tfg_fused_ratio(self._h))

    def export(self):
        """Flat host copy: fields n, tile_size, i_lo[w], i_hi[w], cost[w],
        j_off[w], j_rows[w] (the layout tests compare with schedules_equal)."""
        if self._flat is None:
            fl = _FlatSchedule(self.n, self.tile_size)
            for w in range(2):
                nt, nj = self.num_tiles_per_wave[w], self.num_jrows_per_wave[w]
                ilo = np.zeros(nt + 1, np.int32)
                ihi = np.zeros(nt + 1, np.int32)
                cost = np.zeros(nt + 1, np.float64)
                joff = np.zeros(nt + 1, np.int64)
                jr = np.zeros(nj + 1, np.int32)
                check(lib().tfg_schedule_export(self._h, w, ilo.ctypes.data_as(i32p),
                                                ihi.ctypes.data_as(i32p), cost.ctypes.data_as(f64p),
                                                joff.ctypes.data_as(i64p), jr.ctypes.data_as(i32p)))
                fl.i_lo.append(ilo[:nt])
                fl.i_hi.append(ihi[:nt])
                fl.cost.append(cost[:nt])
                fl.j_off.append(joff)
                fl.j_rows.append(jr[:nj])
            self._flat = fl
        return self._flat

    def wavefronts(self):
        """[[{i_lo, i_hi, j_list, cost}, ...], [...]] like FusedSchedule."""
        fl = self.export()
        out = []
        for w in range(2):
            tiles = []
            for v in range(len(fl.i_lo[w])):
                tiles.append({"i_lo": int(fl.i_lo[w][v]), "i_hi": int(fl.i_hi[w][v]),
                              "j_list": fl.j_rows[w][fl.j_off[w][v]:fl.j_off[w][v + 1]].tolist(),
                              "cost": float(fl.cost[w][v])})
            out.append(tiles)
        return out

    def close(self):
        if self._h and self._h.value:
            lib().tfg_schedule_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class _FlatSchedule:
    n: int
    tile_size: int

    def __post_init__(self):
        self.i_lo, self.i_hi, self.cost, self.j_off, self.j_rows = [], [], [], [], []


def build_schedule(a, cfg: SchedulerConfig, stream=None) -> Schedule:
    """GPU inspector (scheduler.hpp:300-301).  `a` is a host Csr (the
    pattern is copied to HBM) or a DeviceCsr (already resident)."""
    out = C.c_void_p()
    c = cfg.to_c()
    st = _stream_ptr(stream)
    if isinstance(a, DeviceCsr):
        check(lib().tfg_build_schedule(a.n_rows, a.n_cols, a.nnz, a.row_ptr.data_ptr(),
                                       a.col_idx.data_ptr(), C.byref(c), st, C.byref(out)))
    else:
        rp = np.ascontiguousarray(a.row_ptr, np.int32)
        ci = np.ascontiguousarray(a.col_idx, np.int32)
        if ci.size == 0:
            ci = np.zeros(1, np.int32)
        check(lib().tfg_build_schedule_host(a.n_rows, a.n_cols, rp.ctypes.data_as(i32p),
                                            ci.ctypes.data_as(i32p), C.byref(c), st,
                                            C.byref(out)))
    return Schedule(out.value)


def import_schedule(flat) -> Schedule:
    """Upload a flat schedule (e.g. from JSON or another inspector)."""
    nt = (C.c_int64 * 2)(len(flat.i_lo[0]), len(flat.i_lo[1]))
    keep = []

    def arr(a, dt, ptr_t):
        a = np.ascontiguousarray(a, dt)
        if a.size == 0:
            a = np.zeros(1, dt)
        keep.append(a)
        return a.ctypes.data_as(ptr_t)

    ilo = (i32p * 2)(*[arr(flat.i_lo[w], np.int32, i32p) for w in range(2)])
    ihi = (i32p * 2)(*[arr(flat.i_hi[w], np.int32, i32p) for w in range(2)])
    cost = (f64p * 2)(*[arr(flat.cost[w], np.float64, f64p) for w in range(2)])
    joff = (i64p * 2)(*[arr(flat.j_off[w], np.int64, i64p) for w in range(2)])
    jr = (i32p * 2)(*[arr(flat.j_rows[w], np.int32, i32p) for w in range(2)])
    out = C.c_void_p()
    check(lib().tfg_schedule_import(int(flat.n), int(flat.tile_size), nt, ilo, ihi, cost, joff, jr,
                                    C.byref(out)))
    del keep
    return Schedule(out.value)


def fused_ratio_of(sched: Schedule) -> float:
    """scheduler.cpp:247-252."""
    return sched.fused_ratio()


def validate_schedule(a: Csr, sched: Schedule, cfg: SchedulerConfig):
    """scheduler.cpp:254-390 -> (pass, n_violations, over_budget_width1, first_message)."""
    rp = np.ascontiguousarray(a.row_ptr, np.int32)
    ci = np.ascontiguousarray(a.col_idx, np.int32)
    if ci.size == 0:
        ci = np.zeros(1, np.int32)
    c = cfg.to_c()
    ok, nv, ob = C.c_int32(), C.c_int64(), C.c_int64()
    msg = C.create_string_buffer(512)
    check(lib().tfg_validate_schedule(a.n_rows, a.n_cols, rp.ctypes.data_as(i32p),
                                      ci.ctypes.data_as(i32p), sched.handle, C.byref(c),
                                      C.byref(ok), C.byref(nv), C.byref(ob), msg, 512))
    return bool(ok.value), nv.value, ob.value, msg.value.decode()


def checked_schedule(a: Csr, cfg: SchedulerConfig) -> Schedule:
    """bindings.cpp:79-87: build then validate, raising on any violation."""
    s = build_schedule(a, cfg)
    ok, _, _, first = validate_schedule(a, s, cfg)
    if not ok:
        raise RuntimeError("schedule validation failed: " + first)
    return s


# ---- schedule JSON (schedule_io.cpp:9-54) ----------------
def schedule_to_json(sched: Schedule) -> str:
    doc = {"n": sched.n, "tile_size_t": sched.tile_size, "wavefronts": sched.wavefronts(),
           "fused_ratio": sched.fused_ratio()}
    return json.dumps(doc, indent=2) + "\n"


def schedule_from_json(text: str) -> Schedule:
    try:
        root = json.loads(text)
        fl = _FlatSchedule(int(root["n"]), int(root["tile_size_t"]))
        waves = root["wavefronts"]
        if len(waves) != 2:
            raise ValueError("expected exactly 2 wavefronts")
        for wave in waves:
            fl.i_lo.append(np.array([t["i_lo"] for t in wave], np.int32))
            fl.i_hi.append(np.array([t["i_hi"] for t in wave], np.int32))
            fl.cost.append(np.array([t["cost"] for t in wave], np.float64))
            lens = [len(t["j_list"]) for t in wave]
            fl.j_off.append(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64))
            fl.j_rows.append(np.array([j for t in wave for j in t["j_list"]], np.int32))
    except (KeyError, TypeError, json.JSONDecodeError) as e:
        raise RuntimeError(f"schedule json: {e}") from e
    return import_schedule(fl)


# ---------------------------------------------------------------------------
# Device-resident problem + plan (the hot path)
# ---------------------------------------------------------------------------
def _torch():
    import torch

    return torch


def _stream_ptr(stream):
    if stream is None:
        return None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class DeviceCsr:
    """CSR arrays resident in HBM (torch tensors as plain device memory)."""

    def __init__(self, a: Csr, device="cuda", dtype=None):
        torch = _torch()
        self.n_rows, self.n_cols = a.n_rows, a.n_cols
        self.nnz = a.nnz
        vals = a.values if dtype is None else a.values.astype(dtype)
        self.dtype = vals.dtype
        self.row_ptr = torch.from_numpy(a.row_ptr).to(device)
        self.col_idx = torch.from_numpy(a.col_idx if a.nnz else np.zeros(1, np.int32)).to(device)
        self.values = torch.from_numpy(vals if a.nnz else np.zeros(1, vals.dtype)).to(device)

    @property
    def nbytes(self):
        return 4 * (self.n_rows + 1) + self.nnz * (4 + self.dtype.itemsize)


class DeviceProblem:
    """FusedProblem<T> with operands resident in HBM."""

    def __init__(self, a: Csr, b, c: np.ndarray, dtype=np.float64, device="cuda"):
        torch = _torch()
        self.dtype = np.dtype(dtype)
        if not a.square():
            raise ValueError("problem: A must be square")
        self.a = DeviceCsr(a, device, self.dtype)
        self.n = a.n_rows
        c = np.ascontiguousarray(c, self.dtype)
        if isinstance(b, Csr):
            self.b_is_dense = False
            self.b_rows, self.b_cols = b.n_rows, b.n_cols
            # the same host matrix passed as A and B is uploaded once
            self.b = self.a if b is a else DeviceCsr(b, device, self.dtype)
        else:
            b = np.ascontiguousarray(b, self.dtype)
            self.b_is_dense = True
            self.b_rows, self.b_cols = b.shape
            self.b = torch.from_numpy(b).to(device)
        self.c_rows, self.c_cols = c.shape
        self.c = torch.from_numpy(c).to(device)
        self.device = device

    @property
    def b_aliases_a(self) -> bool:
        return self.b is self.a

    def device_inputs(self):
        """The distinct device tensors holding this problem's inputs."""
        ts = [self.a.row_ptr, self.a.col_idx, self.a.values, self.c]
        if self.b_is_dense:
            ts.append(self.b)
        elif not self.b_aliases_a:
            ts += [self.b.row_ptr, self.b.col_idx, self.b.values]
        return ts

    def clone(self):
        """A second device copy of the inputs (for double-buffered streaming)."""
        import copy

        other = copy.copy(self)
        other.a = copy.copy(self.a)
        for name in ("row_ptr", "col_idx", "values"):
            setattr(other.a, name, getattr(self.a, name).clone())
        other.c = self.c.clone()
        if self.b_is_dense:
            other.b = self.b.clone()
        elif self.b_aliases_a:
            other.b = other.a
        else:
            other.b = copy.copy(self.b)
            for name in ("row_ptr", "col_idx", "values"):
                setattr(other.b, name, getattr(self.b, name).clone())
        return other

    def c_struct(self) -> TfgProblem:
        p = TfgProblem()
        p.dtype = _dt_code(self.dtype)
        p.n = self.n
        p.b_is_dense = int(self.b_is_dense)
        p.b_rows, p.b_cols = self.b_rows, self.b_cols
        p.c_rows, p.c_cols = self.c_rows, self.c_cols
        p.a_nnz = self.a.nnz
        p.d_a_row_ptr = self.a.row_ptr.data_ptr()
        p.d_a_col_idx = self.a.col_idx.data_ptr()
        p.d_a_val = self.a.values.data_ptr()
        if self.b_is_dense:
            p.d_b_dense = self.b.data_ptr()
        else:
            p.b_nnz = self.b.nnz
            p.d_b_row_ptr = self.b.row_ptr.data_ptr()
            p.d_b_col_idx = self.b.col_idx.data_ptr()
            p.d_b_val = self.b.values.data_ptr()
        p.d_c = self.c.data_ptr()
        return p


class Plan:
    """Executor plan: schedule bound to a device problem (tfg_plan)."""

    def __init__(self, problem: DeviceProblem, sched: Schedule | None, stream=None,
                 reference_bits: bool = False):
        """reference_bits: grid-stencil SpMM rows use the reference's separately
        rounded multiply and add (bit-identical); default one FMA per term
        (within the north-star tolerance).  tfg.h TFG_PLAN_REFERENCE_BITS."""
        from ._lib import PLAN_REFERENCE_BITS

        self.problem = problem
        self._p = problem.c_struct()
        h = C.c_void_p()
        flags = PLAN_REFERENCE_BITS if reference_bits else 0
        check(lib().tfg_plan_create_ex(C.byref(self._p), sched.handle if sched else None, flags,
                                       0, -1, _stream_ptr(stream), C.byref(h)))
        self._h = h
        sp, fr = C.c_int64(), C.c_int64()
        la, sb = C.c_int32(), C.c_int64()
        check(lib().tfg_plan_info(h, C.byref(sp), C.byref(fr), C.byref(la), C.byref(sb)))
        self.spill_rows, self.fused_rows = sp.value, fr.value
        self.launches, self.scratch_bytes = la.value, sb.value

    def kernels(self) -> dict:
        """Kernel chosen for each stage: {"first_op": ..., "fused": ..., "wave1": ...}."""
        buf = C.create_string_buffer(1024)
        check(lib().tfg_plan_kernels(self._h, buf, 1024))
        return dict(kv.split("=", 1) for kv in buf.value.decode().split())

    def stats(self):
        """RunStats (kernels.hpp:46-50): first_op_rows, second_op_rows, nnz_processed."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().tfg_plan_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"first_op_rows": a.value, "second_op_rows": b.value, "nnz_processed": c.value}

    def execute(self, out=None, stream=None):
        torch = _torch()
        pr = self.problem
        if out is None:
            out = torch.empty((pr.n, pr.c_cols), dtype=getattr(torch, pr.dtype.name),
                              device=pr.device)
        if stream is None:
            stream = torch.cuda.current_stream()
        check(lib().tfg_plan_execute(self._h, C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def execute_from_host(self, host_inputs, device_inputs, out, host_out, stream=None):
        """End-to-end step with host operands: copy each pinned host tensor
        into its HBM twin, execute, copy D back to pinned host memory -- all
        asynchronous on `stream` (the caller synchronises)."""
        torch = _torch()
        if stream is None:
            stream = torch.cuda.current_stream()
        with torch.cuda.stream(stream):
            for h, d in zip(host_inputs, device_inputs):
                d.copy_(h, non_blocking=True)
            self.execute(out, stream)
            host_out.copy_(out, non_blocking=True)
        return host_out

    def profile(self, out=None, stream=None):
        """One execution with per-stage CUDA events: returns
        [(stage, ms, algorithmic_bytes)] for first-op / fused / wavefront-1."""
        torch = _torch()
        pr = self.problem
        if out is None:
            out = torch.empty((pr.n, pr.c_cols), dtype=getattr(torch, pr.dtype.name),
                              device=pr.device)
        if stream is None:
            stream = torch.cuda.current_stream()
        ms = (C.c_double * 3)()
        by = (C.c_int64 * 3)()
        check(lib().tfg_plan_profile(self._h, C.c_void_p(out.data_ptr()), _stream_ptr(stream), ms, by))
        return [(name, ms[k], by[k]) for k, name in enumerate(("first_op", "fused_tiles", "wave1_spmm"))]

    def close(self):
        if self._h and self._h.value:
            lib().tfg_plan_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# By-value API (bindings.cpp:143-191, kernels.hpp:182-236)
# ---------------------------------------------------------------------------
def _require_workers(workers):
    if int(workers) < 1:
        raise ValueError("workers must be >= 1")


def _host_problem(a: Csr, b, c, dtype):
    p = TfgProblem()
    keep = []

    def arr(x, dt):
        x = np.ascontiguousarray(x, dt)
        if x.size == 0:
            x = np.zeros(1, dt)
        keep.append(x)
        return x.ctypes.data

    p.dtype = _dt_code(dtype)
    p.n = a.n_rows
    p.d_a_row_ptr = arr(a.row_ptr, np.int32)
    p.d_a_col_idx = arr(a.col_idx, np.int32)
    p.d_a_val = arr(a.values, dtype)
    p.a_nnz = a.nnz
    if isinstance(b, Csr):
        p.b_is_dense = 0
        p.b_rows, p.b_cols = b.n_rows, b.n_cols
        p.d_b_row_ptr = arr(b.row_ptr, np.int32)
        p.d_b_col_idx = arr(b.col_idx, np.int32)
        p.d_b_val = arr(b.values, dtype)
        p.b_nnz = b.nnz
    else:
        b = np.asarray(b)
        if b.ndim != 2:
            raise ValueError("expected a 2-D array")
        p.b_is_dense = 1
        p.b_rows, p.b_cols = b.shape
        p.d_b_dense = arr(b, dtype)
    c = np.asarray(c)
    if c.ndim != 2:
        raise ValueError("expected a 2-D array")
    p.c_rows, p.c_cols = c.shape
    p.d_c = arr(c, dtype)
    return p, keep


def _check_problem(a: Csr, b, c):
    """problem.check() (kernels.hpp:35-42)."""
    if not a.square():
        raise ValueError("problem: A must be square")
    b_rows = b.n_rows if isinstance(b, Csr) else np.asarray(b).shape[0]
    b_cols = b.n_cols if isinstance(b, Csr) else np.asarray(b).shape[1]
    if b_rows != a.n_cols:
        raise ValueError("problem: B must have n rows")
    if np.asarray(c).shape[0] != b_cols:
        raise ValueError("problem: C rows must match B cols")


def run(a: Csr, b, c, sched: Schedule | None, dtype=None) -> np.ndarray:
    """D = A(BC) through the one-shot host entry (tfg_run_host)."""
    if dtype is None:
        dtype = np.result_type(np.asarray(c).dtype, a.values.dtype)
        if dtype not in (np.float32, np.float64):
            dtype = np.float64
    _check_problem(a, b, c)
    if sched is not None and sched.n != a.n_rows:
        raise ValueError("schedule and problem disagree on n")
    p, keep = _host_problem(a, b, c, dtype)
    d = np.zeros((a.n_rows, np.asarray(c).shape[1]), dtype)
    check(lib().tfg_run_host(C.byref(p), sched.handle if sched else None,
                             C.c_void_p(d.ctypes.data)))
    del keep
    return d


def _config_for(a, b, c, workers, ct_size, cache_words, b_dense, dtype):
    ratio = 0.5 if np.dtype(dtype) == np.float64 else 1.0
    b_cols = b.n_cols if isinstance(b, Csr) else np.asarray(b).shape[1]
    return SchedulerConfig(ct_size=ct_size, num_workers=workers, cache_size_words=cache_words,
                           b_cols=b_cols, c_cols=np.asarray(c).shape[1],
                           index_to_scalar_ratio=ratio, b_is_dense=b_dense)


def fused_gemm_spmm(a: Csr, b, c, workers: int = 1, ct_size: int = 2048,
                    cache_words: int = DEFAULT_CACHE_WORDS, sched: Schedule | None = None,
                    dtype=np.float64) -> np.ndarray:
    """kernels.hpp:182-194 / bindings.cpp:143-157 (B dense)."""
    _require_workers(workers)
    if isinstance(b, Csr):
        raise ValueError("fused_gemm_spmm: B must be dense")
    _check_problem(a, b, c)
    if sched is None:
        cfg = _config_for(a, b, c, workers, ct_size, cache_words, True, np.float64)
        cfg.index_to_scalar_ratio = 0.5  # bindings.cpp:66-77 keeps the default
        sched = checked_schedule(a, cfg)
    return run(a, b, c, sched, dtype)


def fused_spmm_spmm(a: Csr, b: Csr, c, workers: int = 1, ct_size: int = 2048,
                    cache_words: int = DEFAULT_CACHE_WORDS, sched: Schedule | None = None,
                    dtype=np.float64) -> np.ndarray:
    """kernels.hpp:196-208 / bindings.cpp:159-173 (B CSR)."""
    _require_workers(workers)
    if not isinstance(b, Csr):
        raise ValueError("fused_spmm_spmm: B must be sparse")
    _check_problem(a, b, c)
    if sched is None:
        cfg = _config_for(a, b, c, workers, ct_size, cache_words, False, np.float64)
        cfg.index_to_scalar_ratio = 0.5
        sched = checked_schedule(a, cfg)
    return run(a, b, c, sched, dtype)


def unfused_gemm_spmm(a: Csr, b, c, workers: int = 1, dtype=np.float64) -> np.ndarray:
    """kernels.hpp:212-223."""
    _require_workers(workers)
    if isinstance(b, Csr):
        raise ValueError("unfused_gemm_spmm: B must be dense")
    return run(a, b, c, None, dtype)


def unfused_spmm_spmm(a: Csr, b: Csr, c, workers: int = 1, dtype=np.float64) -> np.ndarray:
    """kernels.hpp:225-236."""
    _require_workers(workers)
    if not isinstance(b, Csr):
        raise ValueError("unfused_spmm_spmm: B must be sparse")
    return run(a, b, c, None, dtype)


def gemm(b, c, row_lo: int, row_hi: int, d1: np.ndarray) -> np.ndarray:
    """kernels.hpp:159-169: rows [row_lo, row_hi) of D1 = B*C into d1 (in place), on the GPU."""
    b = np.asarray(b)
    c = np.asarray(c)
    if b.shape[1] != c.shape[0]:
        raise ValueError("gemm: inner dimensions disagree")
    if d1.shape != (b.shape[0], c.shape[1]):
        raise ValueError("gemm: output shape mismatch")
    dt = d1.dtype
    bb = np.ascontiguousarray(b, dt)
    cc = np.ascontiguousarray(c, dt)
    assert d1.flags.c_contiguous
    check(lib().tfg_gemm_rows_host(_dt_code(dt), bb.ctypes.data, b.shape[0], b.shape[1], cc.ctypes.data,
                                   c.shape[0], c.shape[1], int(row_lo), int(row_hi), d1.ctypes.data))
    return d1


def spmm(a: Csr, x, j_list, d: np.ndarray) -> np.ndarray:
    """kernels.hpp:171-180: rows j_list of D = A*X into d (in place), on the GPU."""
    x = np.asarray(x)
    if a.n_cols != x.shape[0]:
        raise ValueError("spmm: inner dimensions disagree")
    if d.shape != (a.n_rows, x.shape[1]):
        raise ValueError("spmm: output shape mismatch")
    dt = d.dtype
    rows = np.ascontiguousarray(j_list, np.int32)
    rr = rows if rows.size else np.zeros(1, np.int32)
    ci = a.col_idx if a.nnz else np.zeros(1, np.int32)
    av = np.ascontiguousarray(a.values, dt) if a.nnz else np.zeros(1, dt)
    xx = np.ascontiguousarray(x, dt)
    assert d.flags.c_contiguous
    check(lib().tfg_spmm_rows_host(_dt_code(dt), a.n_rows, a.n_cols, a.row_ptr.ctypes.data_as(i32p),
                                   ci.ctypes.data_as(i32p), av.ctypes.data, xx.ctypes.data, x.shape[0],
                                   x.shape[1], rr.ctypes.data_as(i32p), rows.size, d.ctypes.data))
    return d


def fused_ratio(a: Csr, tile_size: int) -> float:
    """bindings.cpp:132-141: step-1 fused fraction at a given tile size
    (inspector with p=1 and an unbounded budget, so nothing is split)."""
    cfg = SchedulerConfig(ct_size=int(tile_size), num_workers=1, cache_size_words=2**63 - 1)
    return build_schedule(a, cfg).fused_ratio()


def schedule_json(a: Csr, workers: int = 1, ct_size: int = 2048,
                  cache_words: int = DEFAULT_CACHE_WORDS, b_cols: int = 32, c_cols: int = 32,
                  b_dense: bool = True) -> str:
    """bindings.cpp:118-130."""
    cfg = SchedulerConfig(ct_size=ct_size, num_workers=workers, cache_size_words=cache_words,
                          b_cols=b_cols, c_cols=c_cols, b_is_dense=b_dense)
    return schedule_to_json(checked_schedule(a, cfg))


def device_info():
    arch, sms = C.c_int32(), C.c_int32()
    check(lib().tfg_device_info(C.byref(arch), C.byref(sms)))
    return {"built_arch": arch.value, "sm_count": sms.value}

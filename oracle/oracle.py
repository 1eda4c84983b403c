"""ctypes front-end for the CPU oracle.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this module, and only as the checker or the timed CPU baseline.  The product
package (``paper_2407_00243_b200``) never imports it.

Two back ends share one interface:

* ``Oracle()``   -- ``oracle/liboracle.so``, the plain-C restatement
  (``oracle/tf_oracle.c``) of the reference inspector and executors;
* ``Reference()`` -- ``oracle/_ref/libtfref.so``, the UNMODIFIED reference
  (``/root/reference/proj/src/scheduler.cpp`` + ``include/tilefuse/*.hpp``)
  behind a small extern-"C" shim (``oracle/ref_shim.cpp``).  Built only where
  ``/root/reference`` exists; the built ``.so`` travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libtfref.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class CConfig(C.Structure):
    """tfo_config == tilefuse::SchedulerConfig (scheduler.hpp:15-24)."""

    _fields_ = [
        ("ct_size", C.c_int32),
        ("num_workers", C.c_int32),
        ("cache_size_words", C.c_uint64),
        ("b_cols", C.c_int32),
        ("c_cols", C.c_int32),
        ("index_to_scalar_ratio", C.c_double),
        ("b_is_dense", C.c_int32),
        ("whole_b_cost", C.c_int32),
    ]


class CSchedule(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("tile_size", C.c_int32),
        ("n_tiles", C.c_int64 * 2),
        ("i_lo", i32p * 2),
        ("i_hi", i32p * 2),
        ("cost", f64p * 2),
        ("j_off", i64p * 2),
        ("j_rows", i32p * 2),
    ]


@dataclass
class SchedulerConfig:
    """Python mirror of tilefuse::SchedulerConfig with the reference defaults."""

    ct_size: int = 2048
    num_workers: int = 1
    cache_size_words: int = 160 * 1024
    b_cols: int = 32
    c_cols: int = 32
    index_to_scalar_ratio: float = 0.5
    b_is_dense: bool = True
    whole_b_cost: bool = False

    def to_c(self) -> CConfig:
        return CConfig(
            int(self.ct_size), int(self.num_workers), int(self.cache_size_words),
            int(self.b_cols), int(self.c_cols), float(self.index_to_scalar_ratio),
            int(bool(self.b_is_dense)), int(bool(self.whole_b_cost)))


@dataclass
class OSchedule:
    """Flat two-wavefront schedule (FusedSchedule, scheduler.hpp:39-49)."""

    n: int
    tile_size: int
    i_lo: list = field(default_factory=list)   # [wave] -> int32[n_tiles]
    i_hi: list = field(default_factory=list)
    cost: list = field(default_factory=list)   # float64
    j_off: list = field(default_factory=list)  # int64[n_tiles+1]
    j_rows: list = field(default_factory=list)  # int32

    def n_tiles(self, w: int) -> int:
        return len(self.i_lo[w])

    def tile_j(self, w: int, v: int) -> np.ndarray:
        return self.j_rows[w][self.j_off[w][v]:self.j_off[w][v + 1]]

    def to_c(self):
        """Build a CSchedule view; returns (struct, keepalive)."""
        s = CSchedule()
        s.n = self.n
        s.tile_size = self.tile_size
        keep = []
        for w in range(2):
            arrs = [np.ascontiguousarray(self.i_lo[w], np.int32),
                    np.ascontiguousarray(self.i_hi[w], np.int32),
                    np.ascontiguousarray(self.cost[w], np.float64),
                    np.ascontiguousarray(self.j_off[w], np.int64),
                    np.ascontiguousarray(self.j_rows[w], np.int32)]
            # never hand out NULL for empty arrays
            arrs = [a if a.size else np.zeros(1, a.dtype) for a in arrs]
            keep += arrs
            s.n_tiles[w] = len(self.i_lo[w])
            s.i_lo[w] = arrs[0].ctypes.data_as(i32p)
            s.i_hi[w] = arrs[1].ctypes.data_as(i32p)
            s.cost[w] = arrs[2].ctypes.data_as(f64p)
            s.j_off[w] = arrs[3].ctypes.data_as(i64p)
            s.j_rows[w] = arrs[4].ctypes.data_as(i32p)
        return s, keep


def schedule_from_c(s: CSchedule) -> OSchedule:
    out = OSchedule(int(s.n), int(s.tile_size))
    for w in range(2):
        nt = int(s.n_tiles[w])
        jo = np.ctypeslib.as_array(s.j_off[w], shape=(nt + 1,)).copy()
        tot = int(jo[-1])
        out.i_lo.append(np.ctypeslib.as_array(s.i_lo[w], shape=(nt + 1,))[:nt].copy())
        out.i_hi.append(np.ctypeslib.as_array(s.i_hi[w], shape=(nt + 1,))[:nt].copy())
        out.cost.append(np.ctypeslib.as_array(s.cost[w], shape=(nt + 1,))[:nt].copy())
        out.j_off.append(jo)
        out.j_rows.append(np.ctypeslib.as_array(s.j_rows[w], shape=(tot + 1,))[:tot].copy())
    return out


def schedules_equal(a, b) -> bool:
    """tests/support.hpp:150-165: n, tile size, tile order, i_lo, i_hi,
    j_rows and the exact double cost.  Works on any object exposing the
    OSchedule fields (oracle or GPU export)."""
    if int(a.n) != int(b.n) or int(a.tile_size) != int(b.tile_size):
        return False
    for w in range(2):
        for name in ("i_lo", "i_hi", "j_off", "j_rows"):
            x = np.asarray(getattr(a, name)[w])
            y = np.asarray(getattr(b, name)[w])
            if x.shape != y.shape or not np.array_equal(x.astype(np.int64), y.astype(np.int64)):
                return False
        x = np.asarray(a.cost[w], np.float64)
        y = np.asarray(b.cost[w], np.float64)
        if x.shape != y.shape or not np.array_equal(x.view(np.int64), y.view(np.int64)):
            return False
    return True


def _ptr(a, t):
    return a.ctypes.data_as(t)


class OracleError(ValueError):
    pass


class _Backend:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.lib = C.CDLL(path)
        self.path = path
        L, p = self.lib, self.prefix
        self._f = lambda name: getattr(L, p + name)
        self._f("last_error").restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            msg = self._f("last_error")().decode()
            if rc == 1:
                raise OracleError(msg)
            raise RuntimeError(msg)

    # -- inspector --------------------------------------------------
    def choose_tile_size(self, n, p, ct):
        out = C.c_int32()
        self._check(self._f("choose_tile_size")(C.c_int32(n), C.c_int32(p), C.c_int32(ct), C.byref(out)))
        return out.value

    def step1(self, n_rows, n_cols, row_ptr, col_idx, t):
        rp = np.ascontiguousarray(row_ptr, np.int32)
        ci = np.ascontiguousarray(col_idx, np.int32)
        if ci.size == 0:
            ci = np.zeros(1, np.int32)
        nt = -(-n_rows // t) if t >= 1 and n_rows >= 1 else 1
        off = np.zeros(max(nt, 0) + 2, np.int64)
        jr = np.zeros(max(n_rows, 1), np.int32)
        un = np.zeros(max(n_rows, 1), np.int32)
        nun = C.c_int64()
        self._check(self._f("step1")(C.c_int32(n_rows), C.c_int32(n_cols), _ptr(rp, i32p), _ptr(ci, i32p),
                                     C.c_int32(t), _ptr(off, i64p), _ptr(jr, i32p), _ptr(un, i32p), C.byref(nun)))
        tiles = [jr[off[v]:off[v + 1]].copy() for v in range(nt)]
        return tiles, un[:nun.value].copy()

    def tile_cost(self, n, row_ptr, col_idx, i_lo, i_hi, j_rows, cfg: SchedulerConfig):
        rp = np.ascontiguousarray(row_ptr, np.int32)
        ci = np.ascontiguousarray(col_idx, np.int32)
        if ci.size == 0:
            ci = np.zeros(1, np.int32)
        j = np.ascontiguousarray(j_rows, np.int32)
        jj = j if j.size else np.zeros(1, np.int32)
        out = C.c_double()
        c = cfg.to_c()
        self._check(self._f("tile_cost")(C.c_int32(n), _ptr(rp, i32p), _ptr(ci, i32p), C.c_int32(i_lo),
                                         C.c_int32(i_hi), _ptr(jj, i32p), C.c_int64(j.size), C.byref(c),
                                         C.byref(out)))
        return out.value

    def split_tile(self, n, row_ptr, col_idx, i_lo, i_hi, j_rows, cfg):
        rp = np.ascontiguousarray(row_ptr, np.int32)
        ci = np.ascontiguousarray(col_idx, np.int32)
        if ci.size == 0:
            ci = np.zeros(1, np.int32)
        j = np.ascontiguousarray(j_rows, np.int32)
        jj = j if j.size else np.zeros(1, np.int32)
        s = CSchedule()
        dem = i32p()
        ndem = C.c_int64()
        c = cfg.to_c()
        self._check(self._f("split_tile")(C.c_int32(n), _ptr(rp, i32p), _ptr(ci, i32p), C.c_int32(i_lo),
                                          C.c_int32(i_hi), _ptr(jj, i32p), C.c_int64(j.size), C.byref(c),
                                          C.byref(s), C.byref(dem), C.byref(ndem)))
        pieces = schedule_from_c(s)
        demoted = np.ctypeslib.as_array(dem, shape=(ndem.value + 1,))[:ndem.value].copy()
        self._free_sched(s)
        self._free(dem)
        return pieces, demoted

    def build_schedule(self, n_rows, n_cols, row_ptr, col_idx, cfg: SchedulerConfig):
        rp = np.ascontiguousarray(row_ptr, np.int32)
        ci = np.ascontiguousarray(col_idx, np.int32)
        if ci.size == 0:
            ci = np.zeros(1, np.int32)
        s = CSchedule()
        c = cfg.to_c()
        self._build(n_rows, n_cols, rp, ci, c, s)
        out = schedule_from_c(s)
        self._free_sched(s)
        return out

    def fused_ratio(self, sched: OSchedule) -> float:
        fused = int(sched.j_off[0][-1]) if len(sched.j_off[0]) else 0
        return fused / (2.0 * sched.n) if sched.n >= 1 else 0.0

    def validate_schedule(self, n_rows, n_cols, row_ptr, col_idx, sched: OSchedule, cfg: SchedulerConfig):
        """-> (pass, n_violations, over_budget_width1, first_message)"""
        rp = np.ascontiguousarray(row_ptr, np.int32)
        ci = np.ascontiguousarray(col_idx, np.int32)
        if ci.size == 0:
            ci = np.zeros(1, np.int32)
        cs, keep = sched.to_c()
        c = cfg.to_c()
        nv, ob = C.c_int64(), C.c_int64()
        msg = C.create_string_buffer(512)
        ok = self._f("validate_schedule")(C.c_int32(n_rows), C.c_int32(n_cols), _ptr(rp, i32p), _ptr(ci, i32p),
                                          C.byref(cs), C.byref(c), C.byref(nv), C.byref(ob), msg, C.c_size_t(512))
        del keep
        return bool(ok), nv.value, ob.value, msg.value.decode()

    # -- generators ---------------------------------------------------
    def _csr_out(self, fn, *args):
        rp, ci, v = i32p(), i32p(), f64p()
        self._check(fn(*args, C.byref(rp), C.byref(ci), C.byref(v)))
        return rp, ci, v

    def _take_csr(self, n_rows, rp, ci, v):
        row_ptr = np.ctypeslib.as_array(rp, shape=(n_rows + 1,)).copy()
        nnz = int(row_ptr[-1])
        col_idx = np.ctypeslib.as_array(ci, shape=(nnz + 1,))[:nnz].copy()
        vals = np.ctypeslib.as_array(v, shape=(nnz + 1,))[:nnz].copy()
        for p in (rp, ci, v):
            self._free(p)
        return row_ptr, col_idx, vals

    def gen_random_sparse(self, n, density, seed):
        rp, ci, v = self._csr_out(self._f("gen_random_sparse"), C.c_int32(n), C.c_double(density),
                                  C.c_uint64(seed))
        return self._take_csr(n, rp, ci, v)

    def gen_banded(self, n, hb):
        rp, ci, v = self._csr_out(self._f("gen_banded"), C.c_int32(n), C.c_int32(hb))
        return self._take_csr(n, rp, ci, v)

    def random_dense(self, rows, cols, seed):
        out = np.zeros(max(rows * cols, 1), np.float64)
        self._f("random_dense")(C.c_int32(rows), C.c_int32(cols), C.c_uint64(seed), _ptr(out, f64p))
        return out[:rows * cols].reshape(rows, cols)

    def gen_rect_random(self, rows, cols, density, seed):
        rp, ci, v = self._csr_out(self._f("gen_rect_random"), C.c_int32(rows), C.c_int32(cols),
                                  C.c_double(density), C.c_uint64(seed))
        return self._take_csr(rows, rp, ci, v)


class Oracle(_Backend):
    """The plain-C restatement (oracle/tf_oracle.c)."""

    prefix = "tfo_"

    def __init__(self, path: str = LIB_ORACLE):
        super().__init__(path)
        self._f("fused_ratio").restype = C.c_double

    def _build(self, n_rows, n_cols, rp, ci, c, s):
        self._check(self.lib.tfo_build_schedule(C.c_int32(n_rows), C.c_int32(n_cols), _ptr(rp, i32p),
                                                _ptr(ci, i32p), C.byref(c), C.byref(s)))

    def _free_sched(self, s):
        self.lib.tfo_schedule_free(C.byref(s))

    def _free(self, p):
        self.lib.tfo_free(p)

    def balance(self, rows, weights, num_chunks):
        r = np.ascontiguousarray(rows, np.int32)
        w = np.ascontiguousarray(weights, np.int32)
        rr = r if r.size else np.zeros(1, np.int32)
        ww = w if w.size else np.zeros(1, np.int32)
        off = np.zeros(max(num_chunks, 0) + 2, np.int64)
        self._check(self.lib.tfo_balance(_ptr(rr, i32p), C.c_int64(r.size), _ptr(ww, i32p),
                                         C.c_int64(num_chunks), _ptr(off, i64p)))
        return [r[off[c]:off[c + 1]].copy() for c in range(num_chunks)]

    def mt64(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.lib.tfo_mt64_stream(C.c_uint64(seed), out.ctypes.data_as(C.POINTER(C.c_uint64)), C.c_int64(count))
        return out

    def run(self, n, a, b, c, sched: OSchedule | None, dtype=np.float64, stats=None, workers=0):
        """D = A(BC) with the reference's per-element order.

        a: (row_ptr, col_idx, values); b: dense ndarray (n x bcols) or CSR
        tuple (row_ptr, col_idx, values, n_cols); c: dense ndarray.
        workers=0 -> sequential tfo_run_*, else the OpenMP variant."""
        dt = np.dtype(dtype)
        sfx = "f64" if dt == np.float64 else "f32"
        tp = f64p if dt == np.float64 else C.POINTER(C.c_float)
        arp = np.ascontiguousarray(a[0], np.int32)
        aci = np.ascontiguousarray(a[1], np.int32)
        av = np.ascontiguousarray(a[2], dt)
        aci_ = aci if aci.size else np.zeros(1, np.int32)
        av_ = av if av.size else np.zeros(1, dt)
        cc = np.ascontiguousarray(c, dt)
        if isinstance(b, tuple):
            brp = np.ascontiguousarray(b[0], np.int32)
            bci = np.ascontiguousarray(b[1], np.int32)
            bv = np.ascontiguousarray(b[2], dt)
            bci = bci if bci.size else np.zeros(1, np.int32)
            bv = bv if bv.size else np.zeros(1, dt)
            bcols = int(b[3])
            bd = None
        else:
            brp = bci = bv = None
            bd = np.ascontiguousarray(b, dt)
            bcols = bd.shape[1]
        ccols = cc.shape[1]
        d = np.zeros((n, ccols), dt)
        keep = None
        sp = None
        if sched is not None:
            cs, keep = sched.to_c()
            sp = C.byref(cs)
        st = np.zeros(3, np.int64)
        args = [C.c_int32(n), _ptr(arp, i32p), _ptr(aci_, i32p), _ptr(av_, tp),
                _ptr(brp, i32p) if brp is not None else None,
                _ptr(bci, i32p) if bci is not None else None,
                _ptr(bv, tp) if bv is not None else None,
                _ptr(bd, tp) if bd is not None else None,
                C.c_int32(bcols), _ptr(cc if cc.size else np.zeros(1, dt), tp), C.c_int32(ccols), sp,
                _ptr(d if d.size else np.zeros(1, dt), tp)]
        if workers:
            self._check(getattr(self.lib, f"tfo_run_{sfx}_mt")(*args, C.c_int(workers)))
        else:
            self._check(getattr(self.lib, f"tfo_run_{sfx}")(*args, _ptr(st, i64p)))
        del keep
        if stats is not None:
            stats[:] = st
        return d


class Reference(_Backend):
    """The unmodified reference library (oracle/_ref/libtfref.so)."""

    prefix = "tfr_"

    def __init__(self, path: str = LIB_REF):
        super().__init__(path)
        L = self.lib
        L.tfr_fused_ratio.restype = C.c_double
        L.tfr_problem_create.restype = C.c_void_p
        L.tfr_problem_create.argtypes = [C.c_int, C.c_int32, i32p, i32p, C.c_void_p, i32p, i32p, C.c_void_p,
                                         C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32]
        L.tfr_problem_destroy.argtypes = [C.c_void_p]
        L.tfr_schedule_import.restype = C.c_void_p
        L.tfr_schedule_destroy.argtypes = [C.c_void_p]
        L.tfr_problem_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, i64p, f64p]
        self.libc = C.CDLL(None)
        self.libc.free.argtypes = [C.c_void_p]

    def _build(self, n_rows, n_cols, rp, ci, c, s):
        secs = C.c_double()
        self._check(self.lib.tfr_build_schedule(C.c_int32(n_rows), C.c_int32(n_cols), _ptr(rp, i32p),
                                                _ptr(ci, i32p), C.byref(c), C.byref(s), C.byref(secs)))
        self.last_build_seconds = secs.value

    def _free_sched(self, s):
        for w in range(2):
            for name in ("i_lo", "i_hi", "cost", "j_off", "j_rows"):
                self.libc.free(C.cast(getattr(s, name)[w], C.c_void_p))

    def _free(self, p):
        self.libc.free(C.cast(p, C.c_void_p))

    def balance(self, rows, weights, num_chunks):
        r = np.ascontiguousarray(rows, np.int32)
        w = np.ascontiguousarray(weights, np.int32)
        rr = r if r.size else np.zeros(1, np.int32)
        ww = w if w.size else np.zeros(1, np.int32)
        off = np.zeros(max(num_chunks, 0) + 2, np.int64)
        self._check(self.lib.tfr_balance(_ptr(rr, i32p), C.c_int64(r.size), _ptr(ww, i32p), C.c_int32(w.size),
                                         C.c_int64(num_chunks), _ptr(off, i64p)))
        return [r[off[c]:off[c + 1]].copy() for c in range(num_chunks)]


class RefProblem:
    """A reference FusedProblem<T> held in C++ memory for repeated runs."""

    def __init__(self, ref: Reference, n, a, b, c, dtype=np.float64):
        self.ref = ref
        dt = np.dtype(dtype)
        self.dt = dt
        self.n = n
        self._keep = []

        def k(x, t):
            x = np.ascontiguousarray(x, t)
            if x.size == 0:
                x = np.zeros(1, t)
            self._keep.append(x)
            return x

        arp, aci, av = k(a[0], np.int32), k(a[1], np.int32), k(a[2], dt)
        cc = k(c, dt)
        self.ccols = np.asarray(c).shape[1]
        if isinstance(b, tuple):
            brp, bci, bv = k(b[0], np.int32), k(b[1], np.int32), k(b[2], dt)
            bcols, bd = int(b[3]), None
        else:
            brp = bci = bv = None
            bd = k(b, dt)
            bcols = np.asarray(b).shape[1]
        crows = np.asarray(c).shape[0]
        self.h = ref.lib.tfr_problem_create(
            1 if dt == np.float64 else 0, n, _ptr(arp, i32p), _ptr(aci, i32p), av.ctypes.data,
            _ptr(brp, i32p) if brp is not None else None, _ptr(bci, i32p) if bci is not None else None,
            bv.ctypes.data if bv is not None else None, bd.ctypes.data if bd is not None else None,
            bcols, cc.ctypes.data, crows, self.ccols)
        self._keep = []  # the C++ side copied everything

    def run(self, sched_handle, fused: bool, workers: int, out=True):
        d = np.zeros((self.n, self.ccols), self.dt) if out else None
        st = np.zeros(3, np.int64)
        secs = C.c_double()
        rc = self.ref.lib.tfr_problem_run(self.h, sched_handle, 0 if fused else 1, workers,
                                          d.ctypes.data if d is not None else None, _ptr(st, i64p),
                                          C.byref(secs))
        self.ref._check(rc)
        return d, st, secs.value

    def close(self):
        if self.h:
            self.ref.lib.tfr_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_schedule_handle(ref: Reference, sched: OSchedule):
    cs, keep = sched.to_c()
    h = ref.lib.tfr_schedule_import(C.byref(cs))
    del keep
    return h


def have_reference() -> bool:
    return os.path.exists(LIB_REF)

"""Row-block partitioned D = A(BC) across GPUs.

One process per GPU.  The global schedule (bit-identical to the
reference's) is cut into contiguous row blocks at wavefront-0 tile
boundaries, so every fused row's in-edges are local: wavefront 0 needs no
communication.  Rank r owns rows [lo_r, hi_r): it runs the wavefront-0 tiles
whose i_lo lies in its block and the wavefront-1 rows j in its block.  The one
exchange step is the D1 halo before wavefront 1: the D1 rows r's wavefront-1
rows read but another rank owns, packed by a gather kernel, moved with one
NCCL all-to-all (NVLink/NVSwitch), scattered into r's D1 by global row index.

Inputs (A, B, C) are resident on every rank (each B200 holds 180 GB), so the
halo lists are computed deterministically on every rank from the replicated
pattern and schedule -- no list exchange is needed.

Two drivers share the partition:
* `NativeDistributedPlan` -- the product path, entirely behind the C-ABI
  (include/tfg.h multi-GPU section): cost-balanced cuts
  (tfg_partition_bounds), a device-built halo (tfg_halo_create) that either
  moves the D1 halo with grouped NCCL send/recv while the local-only
  wavefront-1 rows run, or -- GeMM-SpMM, when the cost model says so --
  recomputes the halo rows from the resident B rows; one call per step
  (tfg_plan_execute_dist).  torch.distributed only exchanges the NCCL
  unique id at setup.
* `DistributedPlan` -- the same exchange orchestrated from Python over
  torch.distributed (all_to_all_single); with the NumPy engine of the CPU
  test suite it checks the partition and exchange logic over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def tile_boundaries(flat_sched, n: int, world: int):
    """Row blocks [(lo, hi)] of `world` ranks, cut at wavefront-0 tile starts
    nearest to k*n/world (so fused tiles never straddle ranks)."""
    starts = np.sort(np.asarray(flat_sched.i_lo[0], np.int64))
    if starts.size == 0 or starts[0] != 0:
        starts = np.concatenate([[0], starts])
    cuts = [0]
    for k in range(1, world):
        target = k * n / world
        idx = int(np.searchsorted(starts, target))
        cand = [starts[min(idx, starts.size - 1)], starts[max(idx - 1, 0)]]
        c = int(min(cand, key=lambda x: abs(x - target)))
        cuts.append(max(c, cuts[-1]))
    cuts.append(n)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def owner_of(rows: np.ndarray, bounds) -> np.ndarray:
    his = np.array([hi for _, hi in bounds], np.int64)
    return np.searchsorted(his, rows, side="right")


def wave1_rows(flat_sched) -> np.ndarray:
    return np.asarray(flat_sched.j_rows[1], np.int64)


@dataclass
class HaloPlan:
    """recv[s]: global D1 rows this rank needs from rank s (ascending);
    send[s]: rows this rank sends to rank s."""

    rank: int
    bounds: list
    recv: list
    send: list

    @property
    def recv_rows(self):
        return np.concatenate(self.recv) if self.recv else np.zeros(0, np.int64)

    @property
    def send_rows(self):
        return np.concatenate(self.send) if self.send else np.zeros(0, np.int64)


def halo_needs(row_ptr, col_idx, flat_sched, bounds, rank) -> list:
    """Per peer s: the D1 rows owned by s read by rank's wavefront-1 rows."""
    lo, hi = bounds[rank]
    w1 = wave1_rows(flat_sched)
    mine = w1[(w1 >= lo) & (w1 < hi)]
    rp = np.asarray(row_ptr, np.int64)
    if mine.size:
        lens = rp[mine + 1] - rp[mine]
        idx = np.repeat(rp[mine], lens) + (np.arange(lens.sum()) - np.repeat(np.cumsum(lens) - lens, lens))
        cols = np.unique(np.asarray(col_idx)[idx].astype(np.int64))
    else:
        cols = np.zeros(0, np.int64)
    remote = cols[(cols < lo) | (cols >= hi)]
    own = owner_of(remote, bounds)
    return [remote[own == s] for s in range(len(bounds))]


def halo_plan(row_ptr, col_idx, flat_sched, bounds, rank) -> HaloPlan:
    world = len(bounds)
    recv = halo_needs(row_ptr, col_idx, flat_sched, bounds, rank)
    send = []
    for s in range(world):
        need_s = halo_needs(row_ptr, col_idx, flat_sched, bounds, s)[rank] if s != rank else np.zeros(0, np.int64)
        send.append(need_s)
    return HaloPlan(rank, bounds, recv, send)


class DistributedPlan:
    """Executes one rank's share of the partitioned product.

    engine: stage0(out), stage1(out), gather_d1(rows)->tensor,
            scatter_d1(rows, tensor), device, dtype."""

    def __init__(self, engine, halo: HaloPlan, dist, cols: int):
        import torch

        self.engine = engine
        self.halo = halo
        self.dist = dist
        self.cols = cols
        dev = engine.device
        self.send_idx = torch.as_tensor(halo.send_rows, dtype=torch.int32, device=dev)
        self.recv_idx = torch.as_tensor(halo.recv_rows, dtype=torch.int32, device=dev)
        self.send_splits = [int(x.size) * cols for x in halo.send]
        self.recv_splits = [int(x.size) * cols for x in halo.recv]
        tdt = engine.torch_dtype
        self.recv_buf = torch.empty(max(sum(self.recv_splits), 1), dtype=tdt, device=dev)
        self.halo_rows = int(self.recv_idx.numel())
        self.halo_bytes = self.halo_rows * cols * torch.tensor([], dtype=tdt).element_size()

    def execute(self, out):
        self.engine.stage0(out)
        if self.dist is not None and self.dist.get_world_size() > 1:
            send = self.engine.gather_d1(self.send_idx)
            recv = self.recv_buf[:sum(self.recv_splits)]
            self.dist.all_to_all_single(recv, send.reshape(-1), self.recv_splits, self.send_splits)
            self.engine.scatter_d1(self.recv_idx, recv)
        self.engine.stage1(out)
        return out


class GpuEngine:
    """libtfg partition plan on the current CUDA device."""

    def __init__(self, problem, sched, lo, hi, stream=None, reference_bits=False):
        import ctypes as C

        import torch

        from ._lib import check, lib
        from .tilefuse import _stream_ptr

        self.problem = problem
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.torch_dtype = getattr(torch, problem.dtype.name)
        self._p = problem.c_struct()
        h = C.c_void_p()
        from ._lib import PLAN_REFERENCE_BITS

        check(lib().tfg_plan_create_ex(C.byref(self._p), sched.handle,
                                       PLAN_REFERENCE_BITS if reference_bits else 0, int(lo),
                                       int(hi), _stream_ptr(stream), C.byref(h)))
        self._h = h
        d1 = C.c_void_p()
        check(lib().tfg_plan_d1(h, C.byref(d1)))
        self._d1 = d1.value
        la = C.c_int32()
        check(lib().tfg_plan_info(h, None, None, C.byref(la), None))
        self.launches = la.value
        self._lib, self._check, self._sp = lib, check, _stream_ptr
        self._code = 1 if problem.dtype == np.float64 else 0

    def kernels(self) -> dict:
        """Kernel chosen for each stage of this rank's plan (tfg_plan_kernels)."""
        import ctypes as C

        buf = C.create_string_buffer(256)
        self._check(self._lib().tfg_plan_kernels(self._h, buf, 256))
        return dict(kv.split("=", 1) for kv in buf.value.decode().split())

    def _stream(self):
        import torch

        return self._sp(torch.cuda.current_stream())

    def stage0(self, out):
        import ctypes as C

        self._check(self._lib().tfg_plan_execute_stage(self._h, 0, C.c_void_p(out.data_ptr()), self._stream()))

    def stage1(self, out):
        import ctypes as C

        self._check(self._lib().tfg_plan_execute_stage(self._h, 1, C.c_void_p(out.data_ptr()), self._stream()))

    def gather_d1(self, rows):
        import ctypes as C

        import torch

        cc = self.problem.c_cols
        buf = torch.empty((max(rows.numel(), 1), cc), dtype=self.torch_dtype, device=self.device)
        if rows.numel():
            self._check(self._lib().tfg_gather_rows(self._code, C.c_void_p(self._d1), cc,
                                                    C.c_void_p(rows.data_ptr()), rows.numel(),
                                                    C.c_void_p(buf.data_ptr()), self._stream()))
        return buf[:rows.numel()]

    def scatter_d1(self, rows, data):
        import ctypes as C

        if rows.numel():
            self._check(self._lib().tfg_scatter_rows(self._code, C.c_void_p(data.data_ptr()),
                                                     self.problem.c_cols, C.c_void_p(rows.data_ptr()),
                                                     rows.numel(), C.c_void_p(self._d1), self._stream()))

    def close(self):
        if self._h:
            self._lib().tfg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def owned_output_rows(flat_sched, bounds, rank) -> np.ndarray:
    """Global D rows rank computes: fused rows of its tiles + its wave-1 rows."""
    lo, hi = bounds[rank]
    rows = []
    ilo = np.asarray(flat_sched.i_lo[0])
    for v in np.nonzero((ilo >= lo) & (ilo < hi))[0]:
        rows.append(flat_sched.j_rows[0][flat_sched.j_off[0][v]:flat_sched.j_off[0][v + 1]])
    w1 = wave1_rows(flat_sched)
    rows.append(w1[(w1 >= lo) & (w1 < hi)])
    return np.sort(np.concatenate(rows).astype(np.int64)) if rows else np.zeros(0, np.int64)


# ---------------------------------------------------------------------------
# Native path (C-ABI)
# ---------------------------------------------------------------------------
HALO_AUTO, HALO_EXCHANGE, HALO_RECOMPUTE = 0, 1, 2


def partition_bounds(sched, a, b_cols: int, c_cols: int, dtype, b_is_dense: bool, world: int):
    """tfg_partition_bounds: cuts at wavefront-0 tile starts, balanced by
    estimated bytes per row; returns [(lo, hi)] per rank."""
    import ctypes as C

    from ._lib import check, lib

    rp = np.ascontiguousarray(a.row_ptr, np.int32)
    out = np.zeros(world + 1, np.int32)
    code = 1 if np.dtype(dtype) == np.float64 else 0
    check(lib().tfg_partition_bounds(sched.handle, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                                     int(b_cols), int(c_cols), code, int(b_is_dense), int(world),
                                     out.ctypes.data_as(C.POINTER(C.c_int32))))
    return [(int(out[k]), int(out[k + 1])) for k in range(world)]


def nccl_comm(dist, world: int, rank: int):
    """An NCCL communicator (ncclComm_t as int) from the NCCL the library binds;
    the unique id travels over the torch.distributed group."""
    import ctypes as C

    from ._lib import check, lib

    uid = (C.c_char * 128)()
    if rank == 0:
        check(lib().tfg_nccl_unique_id(uid, 128))
    box = [bytes(uid)]
    if dist is not None and world > 1:
        dist.broadcast_object_list(box, src=0)
    uid = (C.c_char * 128).from_buffer_copy(box[0])
    comm = C.c_void_p()
    check(lib().tfg_nccl_comm_init(int(world), uid, int(rank), C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm):
    from ._lib import check, lib

    import ctypes as C

    check(lib().tfg_nccl_comm_destroy(C.c_void_p(comm)))


class NativeDistributedPlan:
    """One rank of the partitioned product behind the C-ABI."""

    def __init__(self, problem, sched, bounds, rank: int, mode: int = HALO_AUTO, comm=None,
                 stream=None, reference_bits: bool = False):
        import ctypes as C

        from ._lib import PLAN_REFERENCE_BITS, check, lib
        from .tilefuse import _stream_ptr

        self.problem, self.bounds, self.rank, self.comm = problem, bounds, rank, comm
        self.world = len(bounds)
        self._p = problem.c_struct()
        lo, hi = bounds[rank]
        h = C.c_void_p()
        check(lib().tfg_plan_create_ex(C.byref(self._p), sched.handle,
                                       PLAN_REFERENCE_BITS if reference_bits else 0, int(lo),
                                       int(hi), _stream_ptr(stream), C.byref(h)))
        self._plan = h
        b = np.array([lo_ for lo_, _ in bounds] + [bounds[-1][1]], np.int32)
        hh = C.c_void_p()
        check(lib().tfg_halo_create(h, sched.handle, b.ctypes.data_as(C.POINTER(C.c_int32)),
                                    self.world, int(rank), int(mode), _stream_ptr(stream),
                                    C.byref(hh)))
        self._halo = hh
        md, nr, ns = C.c_int32(), C.c_int64(), C.c_int64()
        tx, tr = C.c_double(), C.c_double()
        check(lib().tfg_halo_info(hh, C.byref(md), C.byref(nr), C.byref(ns), C.byref(tx), C.byref(tr)))
        self.mode, self.halo_rows, self.send_rows = md.value, nr.value, ns.value
        self.t_exchange_us, self.t_recompute_us = tx.value, tr.value
        la = C.c_int32()
        check(lib().tfg_plan_info(h, None, None, C.byref(la), None))
        self.launches = la.value + (2 if self.mode == HALO_EXCHANGE else 1)
        self._lib, self._check, self._sp = lib, check, _stream_ptr

    @property
    def mode_name(self):
        return {HALO_EXCHANGE: "exchange", HALO_RECOMPUTE: "recompute"}.get(self.mode, "?")

    def execute(self, out, stream=None):
        import ctypes as C

        import torch

        st = self._sp(stream if stream is not None else torch.cuda.current_stream())
        self._check(self._lib().tfg_plan_execute_dist(self._plan, self._halo,
                                                      C.c_void_p(self.comm) if self.comm else None,
                                                      C.c_void_p(out.data_ptr()), st))
        return out

    def close(self):
        if getattr(self, "_halo", None):
            self._lib().tfg_halo_destroy(self._halo)
            self._halo = None
        if getattr(self, "_plan", None):
            self._lib().tfg_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def execute_emulated(dplans, outs, stream=None):
    """All ranks' steps on one GPU (tfg_plan_execute_dist_emulated)."""
    import ctypes as C

    import torch

    from ._lib import check, lib
    from .tilefuse import _stream_ptr

    w = len(dplans)
    plans = (C.c_void_p * w)(*[d._plan.value for d in dplans])
    halos = (C.c_void_p * w)(*[d._halo.value for d in dplans])
    ds = (C.c_void_p * w)(*[o.data_ptr() for o in outs])
    check(lib().tfg_plan_execute_dist_emulated(plans, halos, w, ds,
                                               _stream_ptr(stream or torch.cuda.current_stream())))

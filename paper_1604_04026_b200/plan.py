"""Device-resident plan: the B200 replacement of the reference's sweep loop.

One ``DevicePlan`` owns, for its lifetime, every device buffer of a
factorization (the ownership rule of SURVEY.md §8(b)): V in both
orientations (CSC uploaded once, CSC of V^T built on the device by
``klnmf_transpose``), the nnz buckets of each side's subproblems, both factors
in the item-major visit-order layout, and (fp32 mode) the maintained
products carried between half-steps.  ``half_step`` is the device version of
``sweep`` (pkg/src/klnmf/solver.py:165-216): fixed-factor row sums
(solver.py:288/294, sparse.py:194-196), then one launch per nnz bucket of the
subproblem solver (_kernels.sweep_range, _kernels.py:123-144).

Precision modes:
  "fp64"  exact mode: fp64 storage, the reference's operation order, no FMA;
          bit-identical to the reference (klnmf_solve_exact).
  "fp32"  throughput mode: fp32 storage of V and the factors, fp64 arithmetic,
          maintained products carried between half-steps (klnmf_solve_fast).

Multi-GPU (torch.distributed, one process per GPU): every rank holds V and
both factors in full; the subproblems of each side (columns for the
F-update, rows for the W-update) are split by a measured device-time model
(``subproblem_cost``): with the fused exchange (fp32 default) the long rows
are dealt across ranks and the rest cut into runs (``dealt_assignment``),
otherwise contiguous cost-balanced ranges (fp32) or nnz-balanced ranges
(fp64).  In fp32 mode the solver kernels store every result into all ranks'
copies through CUDA-IPC mappings (the fused exchange, a barrier before and
after each half-step); otherwise, after each half-step, the updated factor
rows are all-gathered over NCCL.  Results are bitwise independent of the rank count: each
subproblem is solved by exactly one rank with identical inputs, and row sums
are computed from the full replica.

torch is used here only as plumbing: device allocation, the current stream,
and NCCL collectives.  All arithmetic runs in libklnmf.so.
"""

from __future__ import annotations

import ctypes
import dataclasses
import os
import time

import numpy as np
import torch

from . import _lib
from .subproblem import SolveStats, Tolerances

_TIMING = bool(os.environ.get("KLNMF_TIMING"))


class _Ticker:
    """Phase wall times (device-synchronised) when KLNMF_TIMING is set."""

    def __init__(self, what):
        self.what = what
        self.t = time.perf_counter() if _TIMING else 0.0

    def __call__(self, label):
        if _TIMING:
            torch.cuda.synchronize()
            now = time.perf_counter()
            print(f"[klnmf] {self.what}: {label} {1e3 * (now - self.t):.1f} ms", flush=True)
            self.t = now


INT64_MAX = np.iinfo(np.int64).max


def round_rp(r: int) -> int:
    return (r + 3) // 4 * 4


def nnz_balanced_ranges(ptr: np.ndarray, parts: int):
    """Contiguous item ranges [lo, hi) with about equal nnz (atomic items)."""
    ptr = np.asarray(ptr, dtype=np.int64)
    n = ptr.shape[0] - 1
    nnz = int(ptr[-1])
    bounds = [0]
    for q in range(1, parts):
        target = (nnz * q) // parts
        b = int(np.searchsorted(ptr, target, side="left"))
        b = min(max(b, bounds[-1]), n)
        bounds.append(b)
    bounds.append(n)
    return [(bounds[q], bounds[q + 1]) for q in range(parts)]


# Per-entry cost (ns per entry per half-step, one B200) of the fp32 bucket
# kernels by subproblem size, measured at C4 (bench.py kernel table, buckets
# launched one at a time): the warp/block kernels ~0.22-0.26,
# the cluster kernels 0.35 (2 CTAs) to 0.51 (16 CTAs), the cooperative kernel
# 0.48; entries beyond the whole GPU's on-chip capacity (the spill path) cost
# SPILL_NS each.  Every subproblem also pays ITEM_NS of per-coordinate work.
COST_EDGES = np.array([4096, 8192, 16384, 32768, 65536], dtype=np.int64)
COST_NS = np.array([0.24, 0.35, 0.38, 0.44, 0.51, 0.48])
ITEM_NS = 15.0
SPILL_NS = 1.2
ON_CHIP_ENTRIES = 296 * 4096  # cooperative kernel: CTAs x entries per CTA


def spill_scratch_doubles(nnz: int) -> int:
    """Scratch of the long-row kernels' spilled entries: a 32-byte record and
    a one-byte chunk mask per entry of the side (klnmf_solve_args_t.scratch)."""
    return 4 * nnz + (nnz + 7) // 8


def subproblem_cost(sizes: np.ndarray) -> np.ndarray:
    """Modelled device time (ns) of each subproblem of a half-step."""
    sizes = np.asarray(sizes, dtype=np.int64)
    per = COST_NS[np.searchsorted(COST_EDGES, sizes, side="left")]
    spill = np.maximum(sizes - ON_CHIP_ENTRIES, 0)
    return ITEM_NS + per * (sizes - spill) + SPILL_NS * spill


def cost_balanced_ranges(ptr: np.ndarray, parts: int, cost=subproblem_cost):
    """Contiguous item ranges [lo, hi) with about equal modelled device time
    (items atomic).  Balancing by nnz alone hands the first rank the Zipf
    head's long rows, whose per-entry cost is about twice the short ones'."""
    ptr = np.asarray(ptr, dtype=np.int64)
    n = ptr.shape[0] - 1
    if parts <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(parts - 1, 0)
    c = np.concatenate([[0.0], np.cumsum(cost(np.diff(ptr)))])
    bounds = [0]
    for q in range(1, parts):
        b = int(np.searchsorted(c, c[-1] * q / parts, side="left"))
        # the item straddling the target goes to whichever side is closer
        if 0 < b <= n and (c[b] - c[-1] * q / parts) > (c[-1] * q / parts - c[b - 1]):
            b -= 1
        bounds.append(min(max(b, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[q], bounds[q + 1]) for q in range(parts)]


def dealt_assignment(ptr: np.ndarray, parts: int, cost=subproblem_cost, heavy_frac: float = 0.25):
    """Items of each rank (sorted ascending), balancing modelled device time
    when items need not be contiguous (the fused peer exchange stores every
    result by item): items costing more than heavy_frac x the mean rank load
    -- the Zipf head's long rows -- are dealt largest first to the least
    loaded rank; the others are cut, in item order, into runs that fill each
    rank up to the mean."""
    ptr = np.asarray(ptr, dtype=np.int64)
    n = ptr.shape[0] - 1
    if parts <= 1:
        return [np.arange(n, dtype=np.int64)]
    c = cost(np.diff(ptr))
    target = float(c.sum()) / parts
    owner = np.full(n, -1, dtype=np.int64)
    loads = np.zeros(parts)
    heavy = np.nonzero(c > heavy_frac * target)[0]
    for i in heavy[np.argsort(-c[heavy], kind="stable")]:
        q = int(np.argmin(loads))
        owner[i] = q
        loads[q] += c[i]
    light = np.nonzero(owner < 0)[0]
    if light.size:
        room = np.maximum(target - loads, 0.0)
        if room.sum() <= 0.0:
            room = np.ones(parts)
        cl = np.cumsum(c[light])
        cuts = np.searchsorted(cl, np.cumsum(room / room.sum() * cl[-1])[:-1], side="left")
        owner[light] = np.searchsorted(cuts, np.arange(light.size), side="right")
    return [np.nonzero(owner == q)[0] for q in range(parts)]


def _check_fp32_range(V) -> None:
    """fp32 storage of V must keep every (positive) value a normal float:
    below FLT_MIN it would round to 0 or a subnormal (1/v = inf, then NaN in
    the entry state), above FLT_MAX to inf."""
    vals = getattr(V, "values", None)
    if not isinstance(vals, np.ndarray) or vals.size == 0:
        return  # device matrices are generated in fp32 already
    if vals.dtype == np.float64 and vals.flags.c_contiguous:
        lo_c, hi_c = ctypes.c_double(), ctypes.c_double()  # host threads: numpy's min/max took 50 ms at C4
        _lib.call("klnmf_host_minmax_f64", vals.ctypes.data, vals.size, ctypes.byref(lo_c), ctypes.byref(hi_c))
        lo, hi = lo_c.value, hi_c.value
    else:
        lo, hi = float(vals.min()), float(vals.max())
    fi = np.finfo(np.float32)
    if lo < float(fi.tiny) or hi > float(fi.max):
        raise ValueError(f"V values span [{lo:g}, {hi:g}], outside the normal fp32 range "
                         f"[{float(fi.tiny):g}, {float(fi.max):g}]; use precision='fp64'")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


@dataclasses.dataclass
class SidePlan:
    name: str                 # "F" (columns of V) or "W" (rows of V)
    ptr: torch.Tensor         # int64[n_mov+1]
    idx: torch.Tensor         # int32[nnz]
    val: torch.Tensor         # float32/64[nnz]
    n_fix: int
    n_mov: int
    nnz: int
    ptr_host: np.ndarray
    ranges: list | None       # per-rank [lo, hi) (contiguous ownership), or None
    items: torch.Tensor       # int32, this rank's items, sorted by nnz descending
    buckets: list             # [(kernel_id, start, count)], largest first
    tmap: torch.Tensor | None = None  # int32[nnz] entry -> position in the other side
    coop: tuple | None = None  # long-row bucket: (schedule, n_waves, n_ctas, sync, n_groups, spills)
    owned: list | None = None  # per-rank item arrays (dealt ownership), or None

    def owned_items(self, rank: int) -> np.ndarray:
        """Items rank `rank` solves in this side's half-steps."""
        if self.owned is not None:
            return self.owned[rank]
        lo, hi = self.ranges[rank]
        return np.arange(lo, hi, dtype=np.int64)

    def side_struct(self) -> _lib.Side:
        return _lib.Side(self.ptr.data_ptr(), self.idx.data_ptr(), self.val.data_ptr(),
                         self.n_fix, self.n_mov, self.nnz)


class DevicePlan:
    def __init__(self, V, rank: int, precision: str = "fp64", device=None, group=None,
                 ledger=None, fast_kernels: list | None = None, order: str = "shared", order_seed: int = 0,
                 fused_exchange: bool | None = None):
        if precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        if order not in ("shared", "counter"):
            raise ValueError("order must be 'shared' or 'counter'")
        if order == "counter" and precision != "fp32":
            raise ValueError("the counter coordinate order is an fp32-mode option (fp64 is the oracle mode)")
        if precision == "fp32" and round_rp(int(rank)) > 256:
            raise ValueError("the fp32 mode supports rank <= 256 (use precision='fp64' above that)")
        if precision == "fp32" and max(int(V.shape[0]), int(V.shape[1])) * round_rp(int(rank)) >= 2**31 - 1:
            raise ValueError("the fp32 mode needs max(n, m) x padded rank < 2^31 (32-bit gather offsets); "
                             "use precision='fp64' or a smaller rank")
        self.order_mode = _lib.ORDER_COUNTER if order == "counter" else _lib.ORDER_SHARED
        self.order_seed = int(order_seed) & (2**64 - 1) if order == "counter" else 0
        if precision == "fp32":
            _check_fp32_range(V)
        if not torch.cuda.is_available():
            raise RuntimeError("DevicePlan needs a CUDA device (no CPU fallback)")
        _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        self.dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.fp32 = precision == "fp32"
        self.precision = precision
        self.vdt = torch.float32 if self.fp32 else torch.float64
        self.r = int(rank)
        self.rp = round_rp(self.r)
        self.n, self.m = V.shape
        self.nnz = V.nnz
        if self.nnz >= 2**31 - 1:
            raise ValueError("nnz must be < 2^31")
        self.group = group
        if group is not None:
            import torch.distributed as dist
            self.rank_id = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank_id, self.world = 0, 1
        self.ledger = ledger
        dev = self.dev

        tick = _Ticker("plan")
        with torch.cuda.device(dev):
            self.stream_ptr = torch.cuda.current_stream(dev).cuda_stream
            # CSC of V (F-side) uploaded once; CSC of V^T (W-side) built on device
            from .synth import DeviceMatrix

            if isinstance(V, DeviceMatrix):  # already on the device (synth.generate_device)
                col_ptr_host = V.col_ptr_host
                csc_ptr = V.col_ptr.to(dev)
                csc_idx = V.row_idx.to(dev) if self.nnz else torch.empty(1, dtype=torch.int32, device=dev)
                csc_val = V.values.to(dev, self.vdt) if self.nnz else torch.empty(1, dtype=self.vdt, device=dev)
            else:
                col_ptr_host = V.col_ptr
                csc_ptr = torch.from_numpy(V.col_ptr).to(dev)
                csc_idx = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
                csc_val = torch.empty(max(self.nnz, 1), dtype=self.vdt, device=dev)
                row_idx = np.ascontiguousarray(V.row_idx, dtype=np.int64)
                values = np.ascontiguousarray(V.values, dtype=np.float64)
                _lib.call("klnmf_upload_i64_as_i32", row_idx.ctypes.data, self.nnz, csc_idx.data_ptr(),
                          self.stream_ptr)
                _lib.call("klnmf_upload_f64_as_f32" if self.fp32 else "klnmf_upload_f64", values.ctypes.data,
                          self.nnz, csc_val.data_ptr(), self.stream_ptr)
            csr_ptr = torch.empty(self.n + 1, dtype=torch.int64, device=dev)
            csr_idx = torch.empty(self.nnz, dtype=torch.int32, device=dev)
            csr_val = torch.empty(self.nnz, dtype=self.vdt, device=dev)
            map_csr2csc = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
            map_csc2csr = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
            tick("upload V")
            _lib.call("klnmf_transpose", csc_ptr.data_ptr(), csc_idx.data_ptr(), csc_val.data_ptr(),
                      csc_val.element_size(), self.n, self.m, self.nnz, csr_ptr.data_ptr(),
                      csr_idx.data_ptr(), csr_val.data_ptr(), map_csr2csc.data_ptr(),
                      map_csc2csr.data_ptr(), self.stream_ptr)
            csr_ptr_host = csr_ptr.cpu().numpy()

            tick("transpose")
            self.fast_kernels = fast_kernels if fast_kernels is not None else _lib.fast_kernels(self.rp)
            if fused_exchange is None:
                fused_exchange = os.environ.get("KLNMF_FUSED_EXCHANGE", "1") != "0"
            # the fused exchange stores every result by item, so sharded fp32
            # runs may own any item set: long rows are dealt across ranks
            self._dealt = self.world > 1 and self.fp32 and bool(fused_exchange)
            self.sides = {
                "F": self._make_side("F", csc_ptr, csc_idx, csc_val, self.n, self.m, col_ptr_host,
                                     map_csc2csr if self.fp32 else None),
                "W": self._make_side("W", csr_ptr, csr_idx, csr_val, self.m, self.n, csr_ptr_host,
                                     map_csr2csc if self.fp32 else None),
            }
            tick("buckets")
            if self.fp32:
                for sp in self.sides.values():
                    self._build_coop(sp)
            tick("coop schedule")
            self._track("V_csc", csc_ptr, csc_idx, csc_val)
            self._track("V_csr", csr_ptr, csr_idx, csr_val)
            if self.fp32:
                self._track("entry_maps", map_csr2csc, map_csc2csr)
            self.factors = {
                "W": torch.zeros(self.n, self.rp, dtype=self.vdt, device=dev),
                "F": torch.zeros(self.m, self.rp, dtype=self.vdt, device=dev),
            }
            self._track("W", self.factors["W"])
            self._track("F", self.factors["F"])
            self.order = {"W": None, "F": None}  # natural coordinate at each position
            nz = max(self.nnz, 1)
            if self.fp32:
                self.t = {"csc": torch.zeros(nz, dtype=torch.float64, device=dev),
                          "csr": torch.zeros(nz, dtype=torch.float64, device=dev)}
                self._track("t", self.t["csc"], self.t["csr"])
                # scratch backs per-entry state that cannot stay on chip (rows
                # longer than the whole GPU's on-chip capacity, long-row
                # bucket): a 32-byte record per entry
                need_spill = any(s.coop is not None and s.coop[5] for s in self.sides.values())
                self.scratch = torch.empty(spill_scratch_doubles(nz) if need_spill else 4, dtype=torch.float64,
                                           device=dev)
            else:
                self.t = None
                self.scratch = torch.empty(nz, dtype=torch.float64, device=dev)
            self._track("scratch", self.scratch)
            self.t_current = None  # which maintained-product array is valid ("csc"/"csr")
            self.stats = torch.zeros(_lib.STATS_LEN, dtype=torch.int64, device=dev)
            self.sum_pos = torch.zeros(self.rp, dtype=torch.float64, device=dev)
            # rows: perm_in, perm_out, nat_pos, [iteration counter of the counter order]
            self._perm = torch.zeros(4, self.rp, dtype=torch.int32, device=dev)
            self._perm_host = torch.zeros(4, self.rp, dtype=torch.int32).pin_memory()
            self._perm_event = None
            self.use_graphs = True
            # per-row chunk nonzero masks of the fixed factor (long-row kernels; KLNMF_SLICE_MASKS=0: off)
            self.slice_masks = os.environ.get("KLNMF_SLICE_MASKS", "1") != "0"
            self._fixed_mask = torch.zeros(max(self.n, self.m), dtype=torch.int32, device=dev)
            self._track("fixed_mask", self._fixed_mask)
            self._slice_words = None
            if self.fp32 and self.slice_masks and self.r <= 128:
                lanes_of = {k[0]: k[2] for k in self.fast_kernels}
                coop_id = self._stream_kernel_id()
                if any(c > 0 and (kid == coop_id or lanes_of.get(kid, 0) > 256)
                       for sd in self.sides.values() for kid, _, c in sd.buckets):
                    # 8 bytes of mask-word space per entry, only when a side has long rows
                    self._slice_words = torch.empty(4 * max(self.nnz, 1), dtype=torch.int16, device=dev)
                    self._track("slice_words", self._slice_words)
            self._capturing = False
            # streams (and fork/join events) for running independent buckets
            # concurrently; concurrent = False launches them one at a time
            # (per-kernel timing without overlap)
            self.concurrent = True
            self._par_streams = [torch.cuda.Stream(dev) for _ in range(int(os.environ.get("KLNMF_PAR_STREAMS", "6")))]
            self._fork_event = self._new_event()
            self._join_events = [self._new_event() for _ in self._par_streams]
            if self.fp32:
                _lib.call("klnmf_prepare_fast", self.rp)
            self._graphs = {}
            self._uses = {}
            self.graph_after = 2  # uses of a half-step key before its launch sequence is captured
            self._pos = torch.zeros(2, self.rp, dtype=torch.int32, device=dev)
            tick("buffers, prepare")
            # sharded fp32 runs exchange results inside the kernels (peer
            # stores through CUDA IPC) unless disabled; fp64 all-gathers
            self._peers = None
            self._ipc_bases = []
            if self.world > 1 and self.fp32 and fused_exchange:
                self._setup_peers()
                tick("peer mappings")
                if self._peers is None and self._dealt:
                    # the NCCL all-gather moves contiguous ranges: re-split
                    self._dealt = False
                    for name, sp in list(self.sides.items()):
                        self.sides[name] = self._make_side(name, sp.ptr, sp.idx, sp.val, sp.n_fix, sp.n_mov,
                                                           sp.ptr_host, sp.tmap)
                        self._build_coop(self.sides[name])
                    if any(sp.coop is not None and sp.coop[5] for sp in self.sides.values()):
                        self.scratch = torch.empty(spill_scratch_doubles(max(self.nnz, 1)), dtype=torch.float64,
                                                   device=dev)

        # maintained-product layout (klnmf_solve_args_t.t_scatter): each
        # half-step scatters its products into the other side's entry order,
        # so the next half-step reads them coalesced; the all-gather exchange
        # moves contiguous entry ranges and keeps the gathered layout
        self.t_scatter = bool(self.fp32 and (self.world == 1 or self._peers is not None)
                              and os.environ.get("KLNMF_T_SCATTER", "1") != "0")

    def t_orient(self, which: str) -> tuple[str, str]:
        """(read, write) maintained-product arrays of a half-step ("csc" /
        "csr": the entry order each array is stored in)."""
        if self.t_scatter:
            return ("csc", "csr") if which == "F" else ("csr", "csc")
        return ("csr", "csc") if which == "F" else ("csc", "csr")

    def t_entries(self, which: str, name: str) -> torch.Tensor:
        """Maintained products of array `name` in side `which`'s entry order
        (a fresh device tensor)."""
        own = "csc" if which == "F" else "csr"
        t = self.t[name][: self.nnz]
        return t.clone() if name == own else t[self.sides[which].tmap.long()]

    def set_t_entries(self, which: str, name: str, values) -> None:
        """Store products given in side `which`'s entry order into array `name`."""
        own = "csc" if which == "F" else "csr"
        v = torch.as_tensor(values, dtype=torch.float64).to(self.dev)
        if name == own:
            self.t[name][: self.nnz].copy_(v)
        else:
            self.t[name][self.sides[which].tmap.long()] = v

    # ------------------------------------------------------------------
    @staticmethod
    def _new_event():
        h = ctypes.c_void_p()
        _lib.call("klnmf_event_create", ctypes.byref(h))
        return h.value

    def __del__(self):
        for h in [getattr(self, "_fork_event", None), *getattr(self, "_join_events", [])]:
            if h:
                try:
                    _lib.load().klnmf_event_destroy(h)
                except Exception:
                    pass
        bases = getattr(self, "_ipc_bases", [])
        if bases:
            try:
                torch.cuda.synchronize(self.dev)
                for b in bases:
                    _lib.load().klnmf_ipc_close(ctypes.c_void_p(b))
            except Exception:
                pass

    def _setup_peers(self) -> None:
        """Map every other rank's factors and maintained-product arrays
        (CUDA IPC; peer access over NVLink) for the fused exchange: the solver
        kernels store each result into all copies as they produce it
        (klnmf_solve_args_t.peer_*), and a half-step ends with a barrier
        instead of an all-gather.  The values written are the ones the
        all-gather would have moved, so results are bitwise those of the
        all-gather path."""
        import torch.distributed as dist

        bufs = {"W": self.factors["W"], "F": self.factors["F"], "csc": self.t["csc"], "csr": self.t["csr"]}
        mine, error = {}, None
        try:
            for name, ten in bufs.items():
                h = (ctypes.c_char * 64)()
                off = ctypes.c_int64()
                _lib.call("klnmf_ipc_export", ten.data_ptr(), h, ctypes.byref(off))
                mine[name] = (bytes(h), off.value)
        except RuntimeError as exc:
            error = str(exc)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, None if error else mine, group=self.group)
        opened = {}  # one mapping per peer allocation, however many buffers it holds
        peers = {}
        if error is None and all(e is not None for e in everyone):
            try:
                for name in bufs:
                    ptrs = []
                    for q in range(self.world):
                        if q == self.rank_id:
                            continue
                        hb, off = everyone[q][name]
                        if hb not in opened:
                            base = ctypes.c_void_p()
                            _lib.call("klnmf_ipc_open", hb, ctypes.byref(base))
                            opened[hb] = base.value
                        ptrs.append(opened[hb] + off)
                    peers[name] = torch.tensor(ptrs, dtype=torch.int64, device=self.dev)
            except RuntimeError as exc:
                error = str(exc)
        elif error is None:
            error = "a peer rank could not export its buffers"
        # all ranks take the same path: fused only if every rank mapped every peer
        ok = [None] * self.world
        dist.all_gather_object(ok, error is None, group=self.group)
        if not all(ok):
            for b in opened.values():
                try:
                    _lib.call("klnmf_ipc_close", ctypes.c_void_p(b))
                except RuntimeError:
                    pass
            import warnings

            warnings.warn(f"fused peer exchange unavailable ({error or 'on another rank'}); "
                          "falling back to the NCCL all-gather", RuntimeWarning)
            return
        self._ipc_bases = list(opened.values())
        self._peers = peers
        self._barrier_buf = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # every rank has mapped every peer before any kernel stores through a mapping
        dist.barrier(group=self.group)

    @property
    def fused_exchange(self) -> bool:
        return self._peers is not None

    def _peer_barrier(self) -> None:
        """Fused exchange: every rank's work enqueued so far is complete
        before any rank's next work -- after a half-step, so its peer stores
        have landed before anyone reads them; before one, so no peer still
        reads (as the fixed factor, or for the objective) the values about to
        be overwritten in its copy."""
        import torch.distributed as dist

        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._barrier_buf, group=self.group)  # stream-ordered
        else:
            torch.cuda.synchronize(self.dev)
            dist.barrier(group=self.group)

    def _track(self, name, *tensors):
        if self.ledger is not None:
            self.ledger.track(f"dev_{name}", *tensors)

    def _stream_kernel_id(self) -> int:
        for kid, cap, _, _ in self.fast_kernels:
            if cap < 0:
                return kid
        return -1

    def _make_side(self, name, ptr, idx, val, n_fix, n_mov, ptr_host, tmap) -> SidePlan:
        ptr_host = np.asarray(ptr_host, dtype=np.int64)
        ranges, owned = None, None
        if self._dealt:
            owned = dealt_assignment(ptr_host, self.world)
            mine = owned[self.rank_id]
            n_mine = int(mine.size)
        else:
            ranges = (cost_balanced_ranges if self.fp32 else nnz_balanced_ranges)(ptr_host, self.world)
            lo, hi = ranges[self.rank_id]
            n_mine = hi - lo
        if self.fp32:
            caps = [c for _, c, _, _ in self.fast_kernels]
            bounds = np.array([c if c >= 0 else INT64_MAX for c in caps], dtype=np.int64)
            kids = [k for k, _, _, _ in self.fast_kernels]
        else:
            bounds = np.array([INT64_MAX], dtype=np.int64)
            kids = [-1]
        items = torch.empty(max(n_mine, 1), dtype=torch.int32, device=self.dev)
        counts = np.zeros(len(bounds), dtype=np.int64)
        if owned is None:
            _lib.call("klnmf_bucketize", ptr.data_ptr(), lo, hi, bounds.ctypes.data, len(bounds),
                      items.data_ptr(), counts.ctypes.data, self.stream_ptr)
        elif n_mine:
            # the device bucketize's order: size descending, ties by item
            sz = np.diff(ptr_host)[mine]
            order = np.argsort(-sz, kind="stable")
            items.copy_(torch.from_numpy(mine[order].astype(np.int32)))
            counts[:] = np.bincount(np.searchsorted(bounds, sz, side="left"), minlength=len(bounds))
        # items are sorted by nnz descending: the largest bucket comes first
        buckets = []
        start = 0
        for b in range(len(bounds) - 1, -1, -1):
            c = int(counts[b])
            buckets.append((kids[b], start, c))
            start += c
        assert start == n_mine, (start, n_mine)
        return SidePlan(name, ptr, idx, val, int(n_fix), int(n_mov), int(ptr[-1].item()) if n_mov else 0,
                        ptr_host, ranges, items, buckets, tmap, owned=owned)

    def _build_coop(self, sp: SidePlan) -> None:
        """Pack the long-row bucket into waves of the cooperative kernel.

        Each row gets G = ceil(nnz / entries_per_cta) CTAs (capped at the CTA
        count: beyond that its state spills to global memory); rows are taken
        largest first and placed first-fit into waves of n_ctas CTAs."""
        kid = self._stream_kernel_id()
        start, count = next(((st, c) for k, st, c in sp.buckets if k == kid), (0, 0))
        if count == 0:
            return
        per_cta, n_ctas, group_bytes = _lib.coop_info(self.rp)
        lim = int(os.environ.get("KLNMF_COOP_CTAS", "0"))  # experiment knob: fewer CTAs than resident slots
        if lim > 0:
            n_ctas = min(n_ctas, lim)
        rows = sp.items[start:start + count].cpu().numpy()
        sizes = np.diff(sp.ptr_host)[rows]
        waves = []  # [free CTAs, list of (slot, c0, G)]
        for q, sz in enumerate(sizes):
            G = int(min(n_ctas, max(1, -(-int(sz) // per_cta))))
            for w in waves:
                if w[0] >= G:
                    break
            else:
                w = [n_ctas, []]
                waves.append(w)
            w[1].append((q, n_ctas - w[0], G))
            w[0] -= G
        sched = np.full((len(waves), n_ctas, 4), -1, dtype=np.int32)
        for wi, (_, jobs) in enumerate(waves):
            for q, c0, G in jobs:
                for rank in range(G):
                    sched[wi, c0 + rank] = (q, rank, G, q)
        sched_d = torch.from_numpy(sched).to(self.dev)
        sync = torch.empty(count * group_bytes, dtype=torch.uint8, device=self.dev)
        spills = bool(np.any(sizes > n_ctas * per_cta))  # some row exceeds the whole GPU's on-chip capacity
        sp.coop = (sched_d, len(waves), n_ctas, sync, count, spills)

    def _h2d_i32(self, dst: torch.Tensor, arr) -> None:
        host = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32))
        dst.copy_(host, non_blocking=False)

    def _padded(self, perm: np.ndarray) -> np.ndarray:
        out = np.arange(self.rp, dtype=np.int32)
        out[: self.r] = perm
        return out

    # ------------------------------------------------------------------
    def set_factors(self, w: np.ndarray, f: np.ndarray, order: np.ndarray | None = None) -> None:
        """Upload (r, n) / (r, m) fp64 factors, stored in visit order `order`."""
        order = np.arange(self.r) if order is None else np.asarray(order)
        for name, arr, n_items in (("W", w, self.n), ("F", f, self.m)):
            arr = np.ascontiguousarray(arr, dtype=np.float64)
            if arr.shape != (self.r, n_items):
                raise ValueError(f"{name} must have shape {(self.r, n_items)}")
            o = torch.from_numpy(self._padded(order)).to(self.dev)
            if self.fp32:  # narrowed on host threads: half the bytes over PCIe
                src = torch.empty(self.r, n_items, dtype=torch.float32, device=self.dev)
                _lib.call("klnmf_upload_f64_as_f32", arr.ctypes.data, arr.size, src.data_ptr(), self.stream_ptr)
                _lib.call("klnmf_layout_to_device_f32src", src.data_ptr(), self.r, n_items, o.data_ptr(), self.rp,
                          self.factors[name].data_ptr(), self.stream_ptr)
            else:
                src = torch.empty(self.r, n_items, dtype=torch.float64, device=self.dev)
                _lib.call("klnmf_upload_f64", arr.ctypes.data, arr.size, src.data_ptr(), self.stream_ptr)
                _lib.call("klnmf_layout_to_device", src.data_ptr(), self.r, n_items, o.data_ptr(), self.rp,
                          self.factors[name].data_ptr(), 0, self.stream_ptr)
            self.order[name] = np.asarray(order, dtype=np.int64).copy()
        self.t_current = None

    def get_factors(self):
        """Download both factors as (r, n) / (r, m) fp64 numpy arrays."""
        out = []
        for name, n_items in (("W", self.n), ("F", self.m)):
            o = torch.from_numpy(self._padded(self.order[name])).to(self.dev)
            host = np.empty((self.r, n_items), dtype=np.float64)
            if self.fp32:
                # fp32 values cross PCIe and are widened (exactly) on host threads
                dst = torch.empty(self.r, n_items, dtype=torch.float32, device=self.dev)
                _lib.call("klnmf_layout_from_device_f32", self.factors[name].data_ptr(), self.r, n_items,
                          o.data_ptr(), self.rp, dst.data_ptr(), self.stream_ptr)
                _lib.call("klnmf_download_f32_as_f64", dst.data_ptr(), host.size, host.ctypes.data, self.stream_ptr)
            else:
                dst = torch.empty(self.r, n_items, dtype=torch.float64, device=self.dev)
                _lib.call("klnmf_layout_from_device", self.factors[name].data_ptr(), self.r, n_items, o.data_ptr(),
                          self.rp, 0, dst.data_ptr(), self.stream_ptr)
                _lib.call("klnmf_download_f64", dst.data_ptr(), host.size, host.ctypes.data, self.stream_ptr)
            out.append(host)
        return out[0], out[1]

    # ------------------------------------------------------------------
    def row_sums_pos(self, name: str, out: torch.Tensor | None = None) -> torch.Tensor:
        """Row sums of a factor by storage position (fp64, device)."""
        out = self.sum_pos if out is None else out
        fac = self.factors[name]
        n_items = fac.shape[0]
        fn = "klnmf_row_sums_fast" if self.fp32 else "klnmf_row_sums_exact"
        _lib.call(fn, fac.data_ptr(), n_items, self.rp, self.r, out.data_ptr(), self.stream_ptr)
        return out

    def row_sums_natural(self, name: str) -> np.ndarray:
        pos = self.row_sums_pos(name, torch.zeros(self.rp, dtype=torch.float64, device=self.dev))
        pos = pos.cpu().numpy()[: self.r]
        out = np.empty(self.r)
        out[self.order[name]] = pos
        return out

    def _init_t(self, which: str, out: torch.Tensor | None = None) -> None:
        """t at every entry of one orientation = <W_i, F_j> from the stored
        factors (into the maintained products, or into `out`)."""
        side = self.sides["W"] if which == "csr" else self.sides["F"]
        fixed = self.factors["F"] if which == "csr" else self.factors["W"]
        moving = self.factors["W"] if which == "csr" else self.factors["F"]
        fo = self.order["F"] if which == "csr" else self.order["W"]
        mo = self.order["W"] if which == "csr" else self.order["F"]
        self._h2d_i32(self._pos[0], self._padded(np.argsort(fo)))
        self._h2d_i32(self._pos[1], self._padded(np.argsort(mo)))
        s = side.side_struct()
        _lib.call("klnmf_init_t", ctypes.byref(s), fixed.data_ptr(), moving.data_ptr(), self.rp,
                  self._pos[0].data_ptr(), self._pos[1].data_ptr(), self.r,
                  (self.t[which] if out is None else out).data_ptr(), self.stream_ptr)
        if out is None:
            self.t_current = which

    def products_from_factors(self) -> torch.Tensor:
        """fp32 mode: <W_i, F_j> recomputed from the stored factors at every
        entry, in the orientation of the current maintained products (a
        fresh tensor; the carried products are untouched) -- for checking
        the carried t against the factors."""
        if not self.fp32 or self.t_current is None:
            raise RuntimeError("no maintained products are carried (fp32 mode, after a half-step)")
        out = torch.empty_like(self.t[self.t_current])
        self._init_t(self.t_current, out)
        return out

    # kernels launched per outer iteration besides the solver buckets:
    # the fast row sums are two launches per half-step
    aux_launches_per_step = 4

    def half_step(self, which: str, ids, ids_next=None, alpha: float = 0.0, beta: float = 0.0,
                  tol: Tolerances = Tolerances(), sums_pos: np.ndarray | None = None,
                  events: list | None = None, iteration: int | None = None) -> None:
        """Solve every subproblem of one side (which="F": columns, W fixed;
        which="W": rows, F fixed) in place, visiting coordinates in `ids`.

        The moving factor is re-stored in visit order `ids` (F) or `ids_next`
        (W, the next iteration's order; defaults to `ids`).  `sums_pos`
        overrides the device row sums (the public sweep() passes the
        caller's sums, solver.py:165).  With `events` (a list), a CUDA event
        pair around every solver launch is appended as (which, kernel_id,
        start, end); with CUDA graphs the pairs are graph nodes, re-recorded
        by every replay.

        Every pointer of a half-step is fixed for the plan's lifetime; only
        the contents of the visit-order maps (and the row sums) change.  The
        launch sequence of each side is therefore captured once into a CUDA
        graph and replayed, the maps arriving by an asynchronous pinned copy.

        With the counter coordinate order (plan order="counter") `iteration`
        is the counter of the per-subproblem chunk orders (it travels with the
        maps, so the captured graphs stay valid).
        """
        torch.cuda.nvtx.range_push(f"klnmf.half_step.{which}")
        try:
            self._half_step(which, ids, ids_next, alpha, beta, tol, sums_pos, events, iteration)
        finally:
            torch.cuda.nvtx.range_pop()

    def _half_step(self, which, ids, ids_next, alpha, beta, tol, sums_pos, events, iteration) -> None:
        if self.order_mode == _lib.ORDER_COUNTER and iteration is None:
            raise ValueError("the counter coordinate order needs the iteration number")
        if self.fp32 and not tol.eps_div > 0.0:
            raise ValueError("the fp32 mode needs eps_div > 0 (its per-entry state is v/(t+eps_div)); "
                             "use precision='fp64' for eps_div = 0")
        ids = np.asarray(ids, dtype=np.int64)
        fixed_name = "W" if which == "F" else "F"
        if self.order[fixed_name] is None or not np.array_equal(self.order[fixed_name], ids):
            raise RuntimeError(f"fixed factor {fixed_name} is not stored in the visit order")
        o_mov = self.order[which]
        out_order = ids if (which == "F" or ids_next is None) else np.asarray(ids_next, dtype=np.int64)
        perm_in = np.argsort(o_mov)[ids]
        perm_out = np.argsort(out_order)[ids]
        nat_pos = np.argsort(ids)
        it_row = np.zeros(self.rp, dtype=np.int64)
        it_row[0] = 0 if iteration is None else int(iteration) & 0xFFFFFFFF
        self._stage_perms(np.stack([self._padded(perm_in), self._padded(perm_out), self._padded(nat_pos),
                                    it_row.astype(np.uint32).view(np.int32)]))
        dev_sums = sums_pos is None
        if not dev_sums:
            sp = np.zeros(self.rp)
            sp[: self.r] = np.asarray(sums_pos, dtype=np.float64)
            self.sum_pos.copy_(torch.from_numpy(sp))
        if self.fp32:
            need = self.t_orient(which)[0]
            if self.t_current != need:
                self._init_t(need)
        if self._peers is not None:
            self._peer_barrier()
        key = (which, float(alpha), float(beta), tol, dev_sums, events is not None, self.concurrent)
        if self.use_graphs:
            entry = self._graphs.get(key)
            if entry is None:
                entry = self._capture(key)
            if entry is not None:
                graph, evs = entry
                graph.replay()
                if events is not None:
                    events.extend(evs)
            else:
                self._launch(which, alpha, beta, tol, dev_sums, events)
        else:
            self._launch(which, alpha, beta, tol, dev_sums, events)
        if self.fp32:
            self.t_current = self.t_orient(which)[1]
        self.order[which] = np.asarray(out_order, dtype=np.int64).copy()
        if self.world > 1:
            torch.cuda.nvtx.range_push(f"klnmf.exchange.{which}")
            self._exchange(which)
            torch.cuda.nvtx.range_pop()

    def _stage_perms(self, host: np.ndarray) -> None:
        """Visit-order maps -> device through a pinned buffer (no host stall).

        The pinned buffer is reused only after the previous copy completed
        (tracked by an event), so a running copy never sees new contents."""
        if self._perm_event is not None:
            self._perm_event.synchronize()
        self._perm_host.numpy()[...] = host
        self._perm.copy_(self._perm_host, non_blocking=True)
        if self._perm_event is None:
            self._perm_event = torch.cuda.Event()
        self._perm_event.record(torch.cuda.current_stream(self.dev))

    def _capture(self, key):
        """Capture one side's launch sequence into a CUDA graph once the key
        has been used ``graph_after`` times (eager before that: a capture
        costs tens of ms, which only pays off over many replays).  The fp32
        kernels' one-time launch attributes were set at plan construction
        (klnmf_prepare_fast); the exact mode always warms up eagerly once."""
        which, alpha, beta, tol, dev_sums, with_events, _ = key
        uses = self._uses.get(key, 0) + 1
        self._uses[key] = uses
        after = int(os.environ.get("KLNMF_GRAPH_AFTER", self.graph_after))
        if uses < max(after, 1 if self.fp32 else 2):
            return None  # run eagerly this time
        t_start = time.perf_counter() if _TIMING else 0.0
        graph = torch.cuda.CUDAGraph()
        capture_stream = torch.cuda.Stream(self.dev)
        evs: list = []
        saved = self.stream_ptr
        try:
            # capture_begin/end rather than torch.cuda.graph(): the context
            # manager also runs gc.collect() and empty_cache(), which hands
            # every cached block (GBs of plan buffers) back to the driver
            with torch.cuda.stream(capture_stream):
                graph.capture_begin()
                try:
                    self.stream_ptr = capture_stream.cuda_stream
                    self._capturing = True
                    self._launch(which, alpha, beta, tol, dev_sums, evs if with_events else None)
                finally:
                    graph.capture_end()
        except Exception:  # capture unsupported here: stay eager
            self.use_graphs = False
            return None
        finally:
            self.stream_ptr = saved
            self._capturing = False
        self._graphs[key] = (graph, evs)
        if _TIMING:
            print(f"[klnmf] captured {which} half-step graph in {1e3 * (time.perf_counter() - t_start):.1f} ms",
                  flush=True)
        return self._graphs[key]

    def _launch(self, which, alpha, beta, tol, dev_sums, events) -> None:
        """Enqueue one half-step on self.stream_ptr: fixed-factor row sums,
        then one solver launch per non-empty nnz bucket (largest first)."""
        fixed_name = "W" if which == "F" else "F"
        side = self.sides[which]
        if dev_sums:
            self.row_sums_pos(fixed_name)
        a = _lib.SolveArgs()
        a.side = side.side_struct()
        a.fixed = self.factors[fixed_name].data_ptr()
        a.moving = self.factors[which].data_ptr()
        a.sum_pos = self.sum_pos.data_ptr()
        a.perm_in = self._perm[0].data_ptr()
        a.perm_out = self._perm[1].data_ptr()
        a.nat_pos = self._perm[2].data_ptr()
        a.r, a.rp = self.r, self.rp
        a.alpha, a.beta = float(alpha), float(beta)
        a.eps_grad, a.eps_x, a.eps_div = float(tol.eps_grad), float(tol.eps_x), float(tol.eps_div)
        a.inner_cap = int(tol.inner_iter_cap)
        a.stats = self.stats.data_ptr()
        a.scratch = self.scratch.data_ptr()
        a.order_mode = self.order_mode
        a.order_side = 0 if which == "F" else 1
        a.order_seed = self.order_seed
        a.order_iter = self._perm[3].data_ptr()
        if self.fp32:
            t_in, t_out = self.t_orient(which)
            a.tmap = side.tmap.data_ptr()
            a.t_in = self.t[t_in].data_ptr()
            a.t_out = self.t[t_out].data_ptr()
            a.t_scatter = int(self.t_scatter)
            if self._peers is not None:
                a.n_peers = self.world - 1
                a.peer_moving = self._peers[which].data_ptr()
                a.peer_t = self._peers[t_out].data_ptr()
        item_base = side.items.data_ptr()
        lib = _lib.load()
        main = self.stream_ptr
        buckets = [b for b in side.buckets if b[2] > 0]
        coop_kid = self._stream_kernel_id()
        if self._slice_words is not None:
            # chunk nonzero masks of the fixed factor's rows for the long-row
            # kernels (cluster widths have more than 256 lanes): all-zero
            # 16-byte chunks are not gathered
            lanes_of = {k[0]: k[2] for k in self.fast_kernels}
            if any(kid == coop_kid or lanes_of.get(kid, 0) > 256 for kid, _, _ in buckets):
                _lib.call("klnmf_chunk_masks", a.fixed, self.factors[fixed_name].shape[0], self.rp, self.r,
                          self._fixed_mask.data_ptr(), main)
                a.fixed_mask = self._fixed_mask.data_ptr()
                a.slice_words = self._slice_words.data_ptr()
        # the buckets are independent (disjoint outputs, atomic stats) and
        # fork over several streams, so one bucket's last partial wave and
        # the few-subproblem buckets overlap the others;
        # the cooperative long-row kernel is launched first (largest bucket);
        # it runs alongside the other buckets (their blocks fill the SM slots
        # its waves leave free: -0.5 ms per C4 iteration), or alone before
        # them with KLNMF_COOP_CONCURRENT=0
        first = [b for b in buckets if self.fp32 and b[0] == coop_kid]
        if os.environ.get("KLNMF_COOP_CONCURRENT", "1") == "1":
            first = []
        rest = [b for b in buckets if b not in first]
        n_par = min(len(self._par_streams), len(rest)) if (self.fp32 and self.concurrent) else 0
        for q, (kid, start, count) in enumerate(first + rest):
            if q == len(first) and n_par > 1:  # fork
                _lib.call("klnmf_event_record", self._fork_event, main, 0)
                for sp in self._par_streams[:n_par]:
                    _lib.call("klnmf_stream_wait", sp.cuda_stream, self._fork_event)
            sptr = main if (q < len(first) or n_par <= 1) else self._par_streams[(q - len(first)) % n_par].cuda_stream
            a.items = item_base + 4 * start
            a.n_items = count
            ev = self._event_pair(events, sptr)
            if not self.fp32:
                _lib.check(lib.klnmf_solve_exact(ctypes.byref(a), sptr), "klnmf_solve_exact")
            elif kid == coop_kid:
                sched, n_waves, n_ctas, sync, n_groups, _ = side.coop
                _lib.check(lib.klnmf_solve_coop(ctypes.byref(a), sched.data_ptr(), n_waves, n_ctas,
                                                sync.data_ptr(), n_groups, sptr), "klnmf_solve_coop")
            else:
                _lib.check(lib.klnmf_solve_fast(ctypes.byref(a), kid, sptr), "klnmf_solve_fast")
            if ev is not None:
                self._record(ev[1], sptr)
                events.append((which, kid if self.fp32 else -1, ev[0], ev[1]))
        if n_par > 1:  # join
            for i, sp in enumerate(self._par_streams[:n_par]):
                _lib.call("klnmf_event_record", self._join_events[i], sp.cuda_stream, 0)
                _lib.call("klnmf_stream_wait", main, self._join_events[i])

    def _event_pair(self, events, sptr):
        if events is None:
            return None
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        self._record(e0, sptr)
        return e0, e1

    def _record(self, ev: torch.cuda.Event, sptr) -> None:
        """Record on stream sptr; inside a graph capture as an external
        (timing-capable) event node."""
        if ev.cuda_event == 0:
            ev.record(torch.cuda.current_stream(self.dev))  # creates the event handle
        _lib.call("klnmf_event_record", ev.cuda_event, sptr, 1 if self._capturing else 0)

    def _exchange(self, which: str) -> None:
        """All-gather the updated rows of the moving factor (and, in fp32
        mode, the maintained products of the updated entries) -- or, with the
        fused exchange, only wait until every rank's kernels have stored
        theirs into all copies."""
        if self._peers is not None:
            self._peer_barrier()
            return
        side = self.sides[which]
        allgather_ranges(self.factors[which], side.ranges, self.group)
        if self.fp32:
            eranges = [(int(side.ptr_host[lo]), int(side.ptr_host[hi])) for lo, hi in side.ranges]
            assert not self.t_scatter  # ranges are contiguous in this side's entry order
            allgather_ranges(self.t[self.t_orient(which)[1]], eranges, self.group)

    # ------------------------------------------------------------------
    def take_stats(self) -> SolveStats:
        """Read and reset the device counters."""
        arr = self.stats.cpu().numpy()
        self.stats.zero_()
        if self.world > 1:
            # every rank counted only its own subproblems
            import torch.distributed as dist
            nccl = dist.get_backend(self.group) == "nccl"
            t = torch.from_numpy(arr.copy()).to(self.dev if nccl else "cpu")
            dist.all_reduce(t, group=self.group)
            arr = t.cpu().numpy()
        return SolveStats.from_array(arr)

    def objective(self, alpha1=0.0, alpha2=0.0, beta1=0.0, beta2=0.0, eps_div=1e-16, from_factors=False):
        """(kl, total, sparsity_w, sparsity_f) -- full_objective, solver.py:219-234.

        fp32 mode reads the data term from the carried maintained products
        (one streaming pass); ``from_factors=True`` recomputes it from the
        stored factors with an r-dot per nonzero, as the reference does."""
        torch.cuda.nvtx.range_push("klnmf.objective")
        try:
            return self._objective(alpha1, alpha2, beta1, beta2, eps_div, from_factors)
        finally:
            torch.cuda.nvtx.range_pop()

    def _objective(self, alpha1, alpha2, beta1, beta2, eps_div, from_factors):
        data = ctypes.c_double()
        if self.fp32 and self.t_current is not None and not from_factors:
            # fp32 mode carries t = <W_i, F_j> for every entry (all ranks hold all
            # of it after the exchange): one streaming pass over (v, t), summed
            # in V's CSC entry order whichever orientation t is carried in
            side = self.sides["F"]
            tmap = 0 if self.t_current == "csc" else side.tmap.data_ptr()
            _lib.call("klnmf_kl_data_term_t_mapped", side.val.data_ptr(), self.t[self.t_current].data_ptr(), tmap,
                      self.nnz, float(eps_div), ctypes.byref(data), self.stream_ptr)
        else:
            side = self.sides["F"]
            s = side.side_struct()
            wpos = self._padded(np.argsort(self.order["W"]))
            fpos = self._padded(np.argsort(self.order["F"]))
            self._h2d_i32(self._pos[0], wpos)
            self._h2d_i32(self._pos[1], fpos)
            _lib.call("klnmf_kl_data_term_dev", ctypes.byref(s), self.factors["W"].data_ptr(),
                      self.factors["F"].data_ptr(), self.rp, self._pos[0].data_ptr(), self._pos[1].data_ptr(),
                      self.r, int(self.fp32), float(eps_div), ctypes.byref(data), self.stream_ptr)
        kl = float(data.value) + float(self.row_sums_natural("W") @ self.row_sums_natural("F"))
        st = {}
        for name in ("W", "F"):
            out = (ctypes.c_double * 3)()
            fac = self.factors[name]
            _lib.call("klnmf_factor_stats", fac.data_ptr(), fac.shape[0], self.rp, self.r, int(self.fp32),
                      out, self.stream_ptr)
            st[name] = (out[0], out[1], out[2])
        total = kl
        total += 0.5 * alpha1 * st["W"][0]
        total += 0.5 * alpha2 * st["F"][0]
        total += beta1 * st["W"][1]
        total += beta2 * st["F"][1]
        spw = st["W"][2] / (self.r * self.n)
        spf = st["F"][2] / (self.r * self.m)
        return kl, total, spw, spf

    def synchronize(self) -> None:
        torch.cuda.synchronize(self.dev)


def allgather_ranges(buf: torch.Tensor, ranges, group) -> None:
    """In-place all-gather of uneven contiguous first-axis ranges of `buf`.

    Rank q owns rows ranges[q] = (lo, hi); afterwards every rank holds all
    rows.  Padded to the longest range for one all_gather_into_tensor.
    """
    import torch.distributed as dist

    me = dist.get_rank(group)
    world = dist.get_world_size(group)
    maxlen = max(hi - lo for lo, hi in ranges)
    if maxlen == 0:
        return
    tail = tuple(buf.shape[1:])
    # NCCL gathers device memory directly; other backends (gloo: CPU tests,
    # several ranks sharing one GPU) stage through host memory
    stage = buf.is_cuda and dist.get_backend(group) != "nccl"
    dev = torch.device("cpu") if stage else buf.device
    send = torch.zeros((maxlen,) + tail, dtype=buf.dtype, device=dev)
    lo, hi = ranges[me]
    send[: hi - lo] = buf[lo:hi]
    recv = torch.empty((world * maxlen,) + tail, dtype=buf.dtype, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    for q, (lo, hi) in enumerate(ranges):
        if q != me and hi > lo:
            buf[lo:hi] = recv[q * maxlen: q * maxlen + (hi - lo)]

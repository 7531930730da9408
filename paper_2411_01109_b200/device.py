"""Device-resident graph and the torch-level entry points of the B200 kernels.

Everything here takes CUDA tensors, launches on torch's current stream and
returns CUDA tensors; nothing synchronises except graph construction (whose
output sizes are data dependent).  torch provides device memory (the caching
allocator backs every workspace) and streams; all arithmetic happens in
libhalfgnn.so.

HBM layout of a DeviceGraph (N vertices, E edges):
    offsets   int64[N+1]   CSR row offsets          (sparse.py:72-94)
    cols      int32[E]     CSR column ids, rows sorted by (row, col)
    t_offsets int64[N+1]   CSC offsets (transposed CSR, sparse.py:109-120)
    t_cols    int32[E]     CSC row ids
    perm      int32[E]     CSC slot -> CSR edge id (stable, the reference's perm)
    factor tables fp16/fp32[N] and degree-bucketed work units, built lazily.
Features are row-major [rows, F] fp16 (or fp32 in float32 mode).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

from . import _native as nat

DTYPE_CODE = {torch.float16: nat.HG_F16, torch.float32: nat.HG_F32}
MIRROR = {"none": "none", "left": "right", "right": "left", "both": "both"}
DEFAULT_SPLIT_CAP = int(os.environ.get("HG_SPLIT_CAP", "512"))  # edges per work unit (A/B knob)
# hg_spmm folds split rows' carries in the launch itself (last-arriving unit,
# arrival counters; bitwise the follow-up kernel's result).  On the
# degree-sorted graphs (locality_order) it is faster (C3 4.279 -> 4.244 ms,
# C4 11.51 -> 11.45, C5 93.15 -> 92.55); on generated ids it was not (4.419 ->
# 4.438 ms).  HG_FUSED_FOLLOWUP=0 selects the separate follow-up launch.
FUSED_FOLLOWUP = os.environ.get("HG_FUSED_FOLLOWUP", "1") != "0"
# hg_spmm packs: aligned blocks of PACK_ROWS rows with few edges in total, walked
# by one team as one edge stream (hg_schedule_build)
PACK_ROWS = 16
PACKING = os.environ.get("HG_SPMM_PACKS", "1") != "0"  # A/B switch for measurement
# edge budget of a pack (all PACK_ROWS rows together) by output row width
# (>= 256 bytes: wide); 0 packs only all-empty blocks.  A pack is walked by
# one team, so the budget bounds its serial chain (profiles/r01/rowshape)
PACK_EDGES_WIDE = int(os.environ.get("HG_PACK_EDGES_WIDE", "64"))
PACK_EDGES_NARROW = int(os.environ.get("HG_PACK_EDGES_NARROW", "64"))
# packs trade parallelism for shorter dependent chains: only worth it when the
# rows far outnumber the resident teams (Cora / Pubmed-sized graphs lost 3x)
PACK_MIN_ROWS = int(os.environ.get("HG_PACK_MIN_ROWS", str(1 << 20)))
LONG_ROW = 4096   # rows longer than this get a whole CTA in the row-owned softmax/sum kernels
SHORT_ROW = 32    # fast GAT kernels: rows up to this many edges get one thread per head


class _Ptr(ctypes.c_void_p):
    """A device pointer argument that keeps its tensor alive until the C call
    has returned (the kernel is then enqueued), so inline temporaries such as
    `_p(t.contiguous())` cannot be freed and their block handed to the next
    argument's temporary before the launch."""

    __slots__ = ("_keep",)


def _p(t):
    if t is None:
        return None
    ptr = _Ptr(t.data_ptr())
    ptr._keep = t
    return ptr


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype_code(t):
    try:
        return DTYPE_CODE[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}") from None


_WS = {}


class Probe:
    """Launch accounting for the bench: `launches` counts libhalfgnn kernels;
    when `timing` is on, hg_spmm calls are bracketed by CUDA events on the
    launching stream and logged with their algorithmic bytes."""

    launches = 0
    timing = False
    keep = False
    records = []

    @classmethod
    def reset(cls, timing=False, keep=False):
        """keep: also hold each call's (cols, edges, x, F) for gather_ceiling."""
        cls.launches = 0
        cls.timing = timing
        cls.keep = keep
        cls.records = []

    @classmethod
    def summary(cls):
        """(total algorithmic bytes, total seconds, launches) of the timed spmm calls."""
        torch.cuda.synchronize()
        tb = sum(r[2] for r in cls.records)
        ts = sum(r[0].elapsed_time(r[1]) for r in cls.records) / 1e3
        return tb, ts, len(cls.records)

    @classmethod
    def compulsory_per_launch(cls):
        """Mean compulsory DRAM bytes per timed spmm call."""
        return sum(r[3] for r in cls.records) / max(len(cls.records), 1)

    @classmethod
    def l2_ideal_seconds(cls, peak_gbs_by_row_bytes):
        """Seconds the timed spmm calls would take at the measured L2 random-gather
        peak for their row width (tools/l2_gather_peak.py), counting the same
        gather-model bytes; None if a width was not measured."""
        total = 0.0
        for r in cls.records:
            rb, _ = r[5]
            fits = [w for w in peak_gbs_by_row_bytes if w >= rb]
            if not fits:
                return None
            total += r[2] / (peak_gbs_by_row_bytes[min(fits)] * 1e9)
        return total

    @classmethod
    def gather_ceiling(cls, reps=3):
        """Seconds the timed spmm calls' gathers alone take (hg_gather_probe on
        the same column ids, feature buffer and width, X warm in L2 as after
        the producing kernel): the floor those calls could reach.  None when a
        call's row exceeds the probe's 1024 bytes."""
        total = 0.0
        for r in cls.records:
            cols, ne, x, f = r[4]
            row_bytes = -(-f * x.element_size() // 16) * 16
            ld = x.stride(0) * x.element_size()
            if row_bytes > 1024 or ld < row_bytes or ld % 16 or x.data_ptr() % 16:
                return None
            gather_probe(cols, ne, x, row_bytes)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(reps):
                gather_probe(cols, ne, x, row_bytes)
            ev1.record()
            torch.cuda.synchronize()
            total += ev0.elapsed_time(ev1) / 1e3 / reps
        return total


def gather_probe(cols, num_edges, x, row_bytes):
    """hg_gather_probe over cols[:num_edges] into x's rows (measurement only)."""
    sink = workspace(16, x.device)
    nat.call("hg_gather_probe", _p(cols), int(num_edges), _p(x), int(row_bytes),
             x.stride(0) * x.element_size(), _p(sink), _stream())


def compulsory_bytes(n_rows, n_cols, num_edges, f, heads=0, elem=2):
    """Bytes an SpMM must move from/to DRAM at least: the column ids and offsets,
    X read once, Y written once (+ the edge weights): 4E + 8(N+1) + e(F n_cols
    + F n_rows) (+ e E H)."""
    return 4 * num_edges + 8 * (n_rows + 1) + elem * f * (n_cols + n_rows) + elem * num_edges * heads


def spmm_bytes(n_rows, n_cols, num_edges, f, heads=0, elem=2):
    """Gather-model bytes of one SpMM: 4E + 8(N+1) + 2F*E + 2F*N (+2E*H)."""
    return (4 * num_edges + 8 * (n_rows + 1) + elem * f * num_edges + elem * f * n_cols
            + elem * num_edges * heads)


def workspace(nbytes: int, device) -> torch.Tensor | None:
    """Per-(device, stream) scratch from torch's caching allocator, grown on demand.
    Kernels on one stream run in order, so one buffer per stream is safe."""
    if nbytes <= 0:
        return None
    key = (torch.device(device), torch.cuda.current_stream(device).cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("halfgnn operators take CUDA tensors")


# ── graph construction ───────────────────────────────────────────────────


def build_csr(n: int, rows: torch.Tensor, cols: torch.Tensor, want_rows: bool = False):
    """CooGraph.from_edges + coo_to_csr on the GPU (sort + dedup, bit-exact).
    rows/cols: int64 CUDA tensors.  Returns (offsets, cols32, rows64|None)."""
    _require_cuda(rows, cols)
    rows = rows.to(torch.int64).contiguous()
    cols = cols.to(torch.int64).contiguous()
    m = rows.numel()
    if cols.numel() != m:
        raise ValueError("rows/cols must be matching 1-D arrays")
    dev = rows.device
    ws = workspace(nat.size_query("hg_build_csr_workspace", m, n), dev)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out_cols = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    out_rows = torch.empty(max(m, 1), dtype=torch.int64, device=dev) if want_rows else None
    e = ctypes.c_int64(0)
    nat.call("hg_build_csr", _p(rows), _p(cols), m, n, _p(offsets), _p(out_cols), _p(out_rows),
             ctypes.byref(e), _p(ws), 0 if ws is None else ws.numel(), _stream())
    e = int(e.value)
    return offsets, out_cols[:e], (out_rows[:e] if want_rows else None)


_INGEST_ERRORS = {2: "expected 'src dst'", 3: "non-integer vertex id", 4: "negative vertex id"}


def read_bytes_device(path, device="cuda") -> torch.Tensor:
    """A file's bytes as a uint8 tensor in HBM (pinned staging, one copy)."""
    import os

    nbytes = os.path.getsize(path)
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory() if nbytes else torch.empty(0, dtype=torch.uint8)
    if nbytes:
        with open(path, "rb") as fh:
            got = fh.readinto(memoryview(host.numpy()))
        if got != nbytes:
            raise OSError(f"{path}: short read ({got} of {nbytes} bytes)")
    return host.to(device, non_blocking=False)


def load_tensor_device(path, device="cuda") -> torch.Tensor:
    """sparse.load_tensor (HSDT: 16-byte header magic, rows u32, cols u32, mode
    u16, pad; little-endian payload; sparse.py:239-263) straight into HBM: the
    header is checked on the host, the payload moves once through pinned memory."""
    import os
    import struct

    with open(path, "rb") as fh:
        head = fh.read(16)
    if len(head) != 16 or head[:4] != b"HSDT":
        raise ValueError(f"{path}: not a tensor file")
    rows, cols, code = struct.unpack("<IIHxx", head[4:])
    dt = {1: torch.float16, 2: torch.float32}.get(code)
    if dt is None:
        raise ValueError(f"{path}: unknown mode code {code}")
    expect = rows * cols * (2 if code == 1 else 4)
    payload = os.path.getsize(path) - 16
    if payload != expect:
        raise ValueError(f"{path}: payload is {payload} bytes, expected {expect}")
    host = torch.empty(rows * cols, dtype=dt).pin_memory()
    with open(path, "rb") as fh:
        fh.seek(16)
        fh.readinto(memoryview(host.numpy()).cast("B"))
    return host.to(device).view(rows, cols)


def parse_edge_text(text: torch.Tensor, where: str = "<text>"):
    """GPU parse of edge-list text (hg_count_lines + hg_parse_edges): returns
    (rows int64, cols int64, max_id) on the text's device, in file order.
    Raises ValueError("{where}:{line}: ...") like sparse.load_edge_list."""
    _require_cuda(text)
    if text.dtype != torch.uint8 or text.dim() != 1:
        raise ValueError("text must be a 1-D uint8 tensor")
    dev = text.device
    nbytes = text.numel()
    n_lines = ctypes.c_int64(0)
    ws = workspace(nat.size_query("hg_count_lines_workspace", nbytes), dev)
    nat.call("hg_count_lines", _p(text), nbytes, ctypes.byref(n_lines), _p(ws),
             0 if ws is None else ws.numel(), _stream())
    lines = int(n_lines.value)
    ws = workspace(nat.size_query("hg_parse_edges_workspace", nbytes, lines), dev)
    rows = torch.empty(max(lines, 1), dtype=torch.int64, device=dev)
    cols = torch.empty(max(lines, 1), dtype=torch.int64, device=dev)
    res = (ctypes.c_int64 * 4)()
    nat.call("hg_parse_edges", _p(text), nbytes, lines, _p(rows), _p(cols), res, _p(ws),
             0 if ws is None else ws.numel(), _stream())
    Probe.launches += 4
    m, top, bad_line, code = (int(v) for v in res)
    if code == 5:
        raise OverflowError(f"{where}: vertex id does not fit in int64")
    if code:
        raise ValueError(f"{where}:{bad_line}: {_INGEST_ERRORS[code]}")
    return rows[:m], cols[:m], top


def transpose_csr(offsets: torch.Tensor, cols: torch.Tensor, n: int):
    """transpose(g, return_perm=True) on the GPU.  Returns (t_offsets, t_cols, perm)."""
    m = cols.numel()
    dev = offsets.device
    ws = workspace(nat.size_query("hg_transpose_workspace", n, m), dev)
    t_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    t_cols = torch.empty(m, dtype=torch.int32, device=dev)
    perm = torch.empty(m, dtype=torch.int32, device=dev)
    nat.call("hg_transpose", _p(offsets), _p(cols), n, m, _p(t_off), _p(t_cols), _p(perm),
             _p(ws), 0 if ws is None else ws.numel(), _stream())
    return t_off, t_cols, perm


def degree_factors(offsets: torch.Tensor, kind: str, dtype=torch.float16) -> torch.Tensor:
    """kind 'inv' (left/right norms) or 'inv_sqrt' (both), from offsets' degrees."""
    n = offsets.numel() - 1
    out = torch.empty(n, dtype=dtype, device=offsets.device)
    code = nat.FACTOR_INV if kind == "inv" else nat.FACTOR_INV_SQRT
    nat.call("hg_degree_factors", _p(offsets), n, code, DTYPE_CODE[dtype], _p(out), _stream())
    return out


@dataclass
class WorkSchedule:
    """Degree-bucketed work units of one CSR (hg_schedule_build)."""

    units: torch.Tensor       # int32 [U, 4] {row, begin, end, slot}
    split_rows: torch.Tensor  # int32 [S, 4] {row, first_slot, nparts, 0}
    num_slots: int
    split_cap: int
    packs: torch.Tensor | None = None  # int32 [P, 4] {first_row, begin, end, rows}

    @property
    def num_packs(self):
        return 0 if self.packs is None else self.packs.shape[0]

    @property
    def num_units(self):
        return self.units.shape[0]

    def finish_state(self):
        """(arrival counters, slot -> split row) for hg_spmm's fused follow-up
        (None, None without split rows).  The counters start zero and every
        launch leaves them zero; launches sharing them must be stream-ordered."""
        st = getattr(self, "_finish", None)
        if st is None:
            ns = self.split_rows.shape[0]
            if ns == 0:
                st = (None, None)
            else:
                dev = self.split_rows.device
                cnt = torch.zeros(ns, dtype=torch.int32, device=dev)
                slot_split = torch.repeat_interleave(
                    torch.arange(ns, dtype=torch.int32, device=dev),
                    self.split_rows[:, 2].long(), output_size=self.num_slots)
                st = (cnt, slot_split)
            self._finish = st
        return st


def build_schedule(offsets: torch.Tensor, split_cap: int = DEFAULT_SPLIT_CAP,
                   pack_rows: int = 0, pack_edges: int = 0) -> WorkSchedule:
    """pack_rows > 0: aligned blocks of pack_rows rows holding at most
    pack_edges edges become packs (hg_spmm only; the other unit consumers take
    pack_rows = 0)."""
    n = offsets.numel() - 1
    m = int(offsets[-1].item())
    dev = offsets.device
    max_units = n + (m + split_cap - 1) // split_cap
    max_split = max(1, (m + split_cap - 1) // split_cap)
    units = torch.empty((max_units, 4), dtype=torch.int32, device=dev)
    split = torch.empty((max_split, 4), dtype=torch.int32, device=dev)
    max_packs = -(-n // pack_rows) if pack_rows else 0
    packs = torch.empty((max(max_packs, 1), 4), dtype=torch.int32, device=dev)
    ws = workspace(nat.size_query("hg_schedule_workspace", n, m, split_cap), dev)
    counts = (ctypes.c_int64 * 4)()
    nat.call("hg_schedule_build", _p(offsets), n, split_cap, pack_rows, pack_edges, _p(units),
             max_units, _p(split), max_split, _p(packs), max_packs, counts, _p(ws),
             0 if ws is None else ws.numel(), _stream())
    return WorkSchedule(units[: counts[0]], split[: counts[1]], int(counts[2]), split_cap,
                        packs[: counts[3]] if pack_rows else None)


@dataclass
class CsrView:
    """One row-owned CSR operand: local rows, columns index a feature matrix of
    n_cols rows (the full graph, or all-gathered rows of a partition)."""

    offsets: torch.Tensor
    cols: torch.Tensor
    n_rows: int
    n_cols: int
    perm: torch.Tensor | None = None     # for a CSC view: slot -> forward edge id
    _sched: dict = field(default_factory=dict, repr=False)

    @property
    def num_edges(self):
        return self.cols.numel()

    def schedule(self, split_cap: int = DEFAULT_SPLIT_CAP, pack_edges: int = -1) -> WorkSchedule:
        """Work units (cached); pack_edges >= 0: aligned blocks of PACK_ROWS rows
        holding at most pack_edges edges become packs (hg_spmm only)."""
        key = (split_cap, pack_edges)
        s = self._sched.get(key)
        if s is None:
            if pack_edges >= 0:
                s = build_schedule(self.offsets, split_cap, PACK_ROWS,
                                   min(pack_edges, split_cap))
            else:
                s = build_schedule(self.offsets, split_cap)
            self._sched[key] = s
        return s

    def row_ids(self) -> torch.Tensor:
        """int32 local row id per edge (cached; the packed SpMM's row stream)."""
        t = self._sched.get("row_ids")
        if t is None:
            deg = self.offsets[1:] - self.offsets[:-1]
            t = torch.repeat_interleave(
                torch.arange(self.n_rows, device=self.offsets.device, dtype=torch.int32), deg)
            self._sched["row_ids"] = t
        return t

    def row_classes(self, short_max: int = SHORT_ROW, long_min: int = LONG_ROW):
        """(medium, long) int32 row ids: short_max < deg <= long_min, and
        deg > long_min (cached); the rest run one thread per (row, head)."""
        key = ("classes", short_max, long_min)
        t = self._sched.get(key)
        if t is None:
            deg = self.offsets[1:] - self.offsets[:-1]
            med = torch.nonzero((deg > short_max) & (deg <= long_min)).flatten().to(torch.int32)
            t = (med, self.long_rows(long_min))
            self._sched[key] = t
        return t

    def long_rows(self, thresh: int = LONG_ROW) -> torch.Tensor:
        """int32 ids of rows with more than `thresh` edges (cached)."""
        key = ("long", thresh)
        t = self._sched.get(key)
        if t is None:
            deg = self.offsets[1:] - self.offsets[:-1]
            t = torch.nonzero(deg > thresh).flatten().to(torch.int32)
            self._sched[key] = t
        return t


class DeviceGraph:
    """Canonical graph resident in HBM: CSR, CSC + perm, factor tables, schedules."""

    def __init__(self, n: int, offsets: torch.Tensor, cols: torch.Tensor,
                 build_transpose: bool = True):
        self.n = int(n)
        self.offsets = offsets
        self.cols = cols
        self.device = offsets.device
        self.fwd = CsrView(offsets, cols, self.n, self.n)
        self.bwd = None
        if build_transpose:
            t_off, t_cols, perm = transpose_csr(offsets, cols, self.n)
            self.bwd = CsrView(t_off, t_cols, self.n, self.n, perm=perm)
        self._factors = {}
        self._rows = None

    @property
    def num_edges(self):
        return self.cols.numel()

    @property
    def perm(self):
        return self.bwd.perm

    @classmethod
    def from_edge_list(cls, path, num_vertices=None, symmetrize_edges=False, device="cuda",
                       build_transpose=True):
        """load_edge_list (sparse.py:143-177) entirely on the GPU: file bytes to
        HBM, parse, validate, canonicalise; nothing but errors returns to the host."""
        rows, cols, top = parse_edge_text(read_bytes_device(path, device), str(path))
        n = int(num_vertices) if num_vertices is not None else top + 1
        if n <= 0:
            raise ValueError(f"{path}: empty graph and no vertex count given")
        if rows.numel() and top >= n:
            bad = int(torch.nonzero((rows >= n) | (cols >= n))[0, 0])
            raise ValueError(f"{path}: vertex id out of range at edge {bad}")
        if symmetrize_edges:
            rows, cols = torch.cat([rows, cols]), torch.cat([cols, rows])
        offsets, c32, _ = build_csr(n, rows, cols)
        return cls(n, offsets, c32, build_transpose=build_transpose)

    @classmethod
    def from_edges(cls, n, rows, cols, device="cuda", build_transpose=True):
        """Canonicalise an arbitrary edge list (any order, duplicates allowed) on the GPU."""
        rows = torch.as_tensor(rows, dtype=torch.int64).to(device)
        cols = torch.as_tensor(cols, dtype=torch.int64).to(device)
        offsets, c32, _ = build_csr(n, rows, cols)
        return cls(n, offsets, c32, build_transpose)

    def rows(self) -> torch.Tensor:
        """int64 row id per CSR edge (csr_to_coo)."""
        if self._rows is None:
            deg = self.offsets[1:] - self.offsets[:-1]
            self._rows = torch.repeat_interleave(
                torch.arange(self.n, device=self.device, dtype=torch.int64), deg)
        return self._rows

    def factor(self, kind: str, side: str, dtype=torch.float16) -> torch.Tensor:
        """Degree factor table; side 'row' uses CSR degrees, 'col' CSC degrees."""
        key = (kind, side, dtype)
        t = self._factors.get(key)
        if t is None:
            offs = self.offsets if side == "row" else self.bwd.offsets
            t = degree_factors(offs, kind, dtype)
            self._factors[key] = t
        return t

    def norm_tables(self, norm: str, transpose: bool, dtype):
        """(in_scale, out_factor) of `norm` for the graph actually traversed
        (the transpose when transpose=True), as kernels._degree_factors does."""
        kind = "inv_sqrt" if norm == "both" else "inv"
        row_side, col_side = ("col", "row") if transpose else ("row", "col")
        fin = self.factor(kind, col_side, dtype) if norm in ("left", "both") else None
        fout = self.factor(kind, row_side, dtype) if norm in ("right", "both") else None
        return fin, fout

    def view(self, transpose: bool = False) -> CsrView:
        if transpose and self.bwd is None:
            raise ValueError("graph was built without its transpose")
        return self.bwd if transpose else self.fwd

    def relabel(self, order: torch.Tensor) -> "DeviceGraph":
        """The same graph with vertex order[i] renamed i (order: new -> old id,
        a permutation); edges, degrees and every per-vertex quantity follow
        their vertex, CSR / CSC rebuilt canonical on the GPU."""
        order = order.to(self.device, torch.int64)
        if order.numel() != self.n:
            raise ValueError("order must be a permutation of the vertices")
        new_of_old = torch.empty_like(order)
        new_of_old[order] = torch.arange(self.n, device=self.device)
        return DeviceGraph.from_edges(self.n, new_of_old[self.rows()],
                                      new_of_old[self.cols.long()], device=self.device,
                                      build_transpose=self.bwd is not None)


def locality_order(offsets, t_offsets=None, parts: int = 1) -> torch.Tensor:
    """Vertex relabelling for gather locality (new -> old id): vertices by
    descending total degree, so the rows that the aggregations gather most
    share L2 lines and DRAM pages (random ids spread each hot 100-256-byte row
    over lines shared with cold rows).  With parts > 1 the sorted vertices are
    dealt round-robin to the parts' contiguous id ranges (each rank of a row
    partition gets an equal share of the hubs, ids degree-sorted inside it).
    Stable, deterministic.  Measured on one B200 (tools/exp/reorder_probe.py):
    C4 F=112 SpMM 4.95 -> 4.32 ms, C5 F=128 13.7 -> 11.2 ms."""
    deg = offsets[1:] - offsets[:-1]
    if t_offsets is not None:
        deg = deg + (t_offsets[1:] - t_offsets[:-1])
    by_deg = torch.argsort(deg, descending=True, stable=True)
    if parts <= 1:
        return by_deg
    n = by_deg.numel()
    k = torch.arange(n, device=by_deg.device)
    # rank p takes sorted positions p, p + parts, ...; ranks laid out in id order
    key = (k % parts) * n + k // parts
    return by_deg[torch.argsort(key, stable=True)]


# ── SpMM ─────────────────────────────────────────────────────────────────


def _row_strided(t):
    """2-D tensor whose rows may be padded (unit column stride)."""
    return t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]


def spmm_csr(view: CsrView, x: torch.Tensor, w=None, w_index=None, heads: int = 1,
             scaling: str = "post", fin=None, fout=None, out=None,
             split_cap: int = DEFAULT_SPLIT_CAP, relu: bool = False, w2_off: int = 0,
             out2=None, combine=None, head_dots=None) -> torch.Tensor:
    """fp32-guarded row-owned SpMM over one CSR view (hg_spmm).  x and out may
    be column slices of wider row-major storage (row strides passed through).
    combine = (res [n_rows, F], ope (device scalar or None), lam): the row store
    writes rnd(rnd(res * ope) + rnd(y * lam)) (GIN's combine; ope None and
    lam 1: a rounded residual add).  head_dots = (g_l, g_r [n_rows, heads],
    a_l, a_r [F]): the row store adds the GAT head-dot backward's dz term,
    rnd(y + rnd(rnd(g_l a_l) + rnd(g_r a_r))) per head (hg_head_dots_bwd's)."""
    _require_cuda(x)
    if not _row_strided(x) or fin is not None:
        x = x.contiguous()
    if x.dim() != 2 or x.shape[0] != view.n_cols:
        raise ValueError(f"feature tensor has {x.shape[0]} rows for {view.n_cols} columns")
    f = x.shape[1]
    dt = _dtype_code(x)
    pack_edges = -1
    if PACKING and view.n_rows >= PACK_MIN_ROWS:
        pack_edges = PACK_EDGES_WIDE if f * x.element_size() >= 256 else PACK_EDGES_NARROW
    sched = view.schedule(split_cap, pack_edges)
    if out is None:
        out = torch.empty((view.n_rows, f), dtype=x.dtype, device=x.device)
    elif not _row_strided(out) or out.shape != (view.n_rows, f) or out.dtype != x.dtype:
        raise ValueError("out must be [n_rows, F] with unit column stride")
    fin_state = sched.finish_state() if FUSED_FOLLOWUP else (None, None)
    nbytes = nat.size_query("hg_spmm_workspace", view.n_cols, f, sched.num_slots,
                            int(fin is not None), heads if out2 is not None else 0, dt)
    ws = workspace(nbytes, x.device)
    w_ld = 0
    if w is not None:
        if w.dim() == 2 and w.stride(1) == 1:
            w_ld = w.stride(0)  # row-strided weights (e.g. interleaved alpha | d_e rows)
        else:
            w = w.contiguous()
        if w.dtype != x.dtype:
            raise ValueError("edge weights must match the feature dtype")
    if Probe.timing:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    c_res = c_ope = None
    c_lam = 1.0
    if combine is not None:
        c_res, c_ope, c_lam = combine
        if c_res.shape != (view.n_rows, f) or c_res.dtype != x.dtype or c_res.stride(1) != 1:
            raise ValueError("combine residual must be [n_rows, F] of the feature dtype")
        if c_ope is not None:
            c_ope = c_ope.reshape(-1)[:1].contiguous()
    hd = (None, None, None, None)
    if head_dots is not None:
        # (head vectors re-based to 32-byte alignment for the store's vector loads)
        hd = tuple(t.to(x.dtype).contiguous() for t in head_dots)
        hd = hd[:2] + tuple(t if t.data_ptr() % 32 == 0 else t.clone() for t in hd[2:])
        if (hd[0].shape != (view.n_rows, heads) or hd[1].shape != (view.n_rows, heads)
                or hd[2].numel() != f or hd[3].numel() != f):
            raise ValueError("head_dots: g_l, g_r [n_rows, heads] and a_l, a_r [F]")
    nat.call("hg_spmm", _p(view.offsets), _p(view.cols), view.n_rows, view.n_cols,
             view.num_edges, _p(sched.units), sched.num_units, _p(sched.split_rows),
             sched.split_rows.shape[0], sched.num_slots, _p(sched.packs), sched.num_packs,
             _p(view.row_ids() if sched.num_packs else None), _p(w), _p(w_index), heads, _p(x),
             _p(out), f, x.stride(0), out.stride(0), nat.SCALING_CODES[scaling], int(relu),
             _p(fin), _p(fout), w_ld, int(w2_off), _p(out2), dt, _p(ws),
             0 if ws is None else ws.numel(), _stream(), *map(_p, fin_state), _p(c_res),
             0 if c_res is None else c_res.stride(0), _p(c_ope), float(c_lam), *map(_p, hd))
    Probe.launches += int(sched.num_units > 0) + int(sched.num_packs > 0) + int(
        sched.split_rows.shape[0] > 0 and fin_state[0] is None) + int(fin is not None)
    if Probe.timing:
        ev1.record()
        Probe.records.append((ev0, ev1, spmm_bytes(view.n_rows, view.n_cols, view.num_edges, f,
                                                   heads if w is not None else 0,
                                                   x.element_size()),
                              compulsory_bytes(view.n_rows, view.n_cols, view.num_edges, f,
                                               heads if w is not None else 0,
                                               x.element_size()),
                              (view.cols, view.num_edges, x, f) if Probe.keep else None,
                              (-(-f * x.element_size() // 16) * 16, view.num_edges)))
    return out


def spmm_csr_acc(view: CsrView, x: torch.Tensor, acc_in=None, acc_out=None, scaling="post",
                 fout=None, out=None, relu=False, split_cap: int = DEFAULT_SPLIT_CAP,
                 w=None, w_index=None, heads: int = 1):
    """One column block of a blocked aggregation (hg_spmm_acc): rows start from
    the fp32 acc_in (None: 0); with acc_out the unrounded fp32 sums go there
    (may be acc_in), else the rows are finished into `out` (returned).  w /
    w_index / heads: edge weights as spmm_csr (w_index maps the block's edges
    to rows of w)."""
    _require_cuda(x)
    if not _row_strided(x):
        x = x.contiguous()
    if x.dim() != 2 or x.shape[0] != view.n_cols:
        raise ValueError(f"feature tensor has {x.shape[0]} rows for {view.n_cols} columns")
    f = x.shape[1]
    dt = _dtype_code(x)
    for a in (acc_in, acc_out):
        if a is not None and (a.dtype != torch.float32 or a.shape != (view.n_rows, f)
                              or not a.is_contiguous()):
            raise ValueError("accumulators must be contiguous float32 [n_rows, F]")
    pack_edges = -1
    if PACKING and view.n_rows >= PACK_MIN_ROWS:
        pack_edges = PACK_EDGES_WIDE if f * x.element_size() >= 256 else PACK_EDGES_NARROW
    sched = view.schedule(split_cap, pack_edges)
    if acc_out is None and out is None:
        out = torch.empty((view.n_rows, f), dtype=x.dtype, device=x.device)
    nbytes = nat.size_query("hg_spmm_workspace", view.n_cols, f, sched.num_slots, 0, 0, dt)
    ws = workspace(nbytes, x.device)
    w_ld = 0
    if w is not None:
        if w.dim() == 2 and w.stride(1) == 1:
            w_ld = w.stride(0)
        else:
            w = w.contiguous()
        if w.dtype != x.dtype:
            raise ValueError("edge weights must match the feature dtype")
    nat.call("hg_spmm_acc", _p(view.offsets), _p(view.cols), view.n_rows, view.n_cols,
             view.num_edges, _p(sched.units), sched.num_units, _p(sched.split_rows),
             sched.split_rows.shape[0], sched.num_slots, _p(sched.packs), sched.num_packs,
             _p(view.row_ids() if sched.num_packs else None), _p(w), _p(w_index), heads, w_ld,
             _p(x), _p(out), f, x.stride(0),
             f if out is None else out.stride(0), nat.SCALING_CODES[scaling], int(relu), _p(fout),
             _p(acc_in), _p(acc_out), dt, _p(ws), 0 if ws is None else ws.numel(), _stream())
    Probe.launches += int(sched.num_units > 0) + int(sched.num_packs > 0) + int(
        sched.split_rows.shape[0] > 0)
    return acc_out if acc_out is not None else out


def spmm(dg: DeviceGraph, x, w=None, scaling="post", norm="none", transpose=False, heads=1,
         out=None, weight_via_perm=False, relu=False, combine=None):
    """SpMMv / SpMMve on the graph (or its transpose), fp32-guarded.
    weight_via_perm: w is indexed by forward edge id and read through perm
    (spmm_weighted backward, models.py:309-311) without materialising w[perm]."""
    view = dg.view(transpose)
    fin, fout = dg.norm_tables(norm, transpose, x.dtype)
    widx = view.perm if (w is not None and weight_via_perm) else None
    return spmm_csr(view, x, w, widx, heads, scaling, fin, fout, out, relu=relu,
                    combine=combine)


def spmm_edge_ref(dg: DeviceGraph, x, w=None, scaling="post", norm="none", transpose=False,
                  warp_chunk=128, warps_per_cta=4, staging=False):
    """Reference-order SpMM (bit-exact with halfsparse.kernels.spmm_v / spmm_ve).
    Returns y, or (y, staging_rows int64, staging_partials) when staging=True."""
    view = dg.view(transpose)
    _require_cuda(x)
    x = x.contiguous()
    f = x.shape[1]
    dt = _dtype_code(x)
    fin, fout = dg.norm_tables(norm, transpose, x.dtype)
    y = torch.empty((view.n_rows, f), dtype=x.dtype, device=x.device)
    m = view.num_edges
    nw = (m + warp_chunk - 1) // warp_chunk
    nc = (nw + warps_per_cta - 1) // warps_per_cta
    st_rows = st_vals = None
    if staging:
        st_rows = torch.empty(max(nc, 1), dtype=torch.int64, device=x.device)
        st_vals = torch.empty((max(nc, 1), f), dtype=x.dtype, device=x.device)
    nbytes = nat.size_query("hg_spmm_edge_ref_workspace", view.n_cols, m, f, warp_chunk,
                            warps_per_cta, int(fin is not None), dt)
    ws = workspace(nbytes, x.device)
    if w is not None:
        w = w.contiguous()
    nat.call("hg_spmm_edge_ref", _p(view.offsets), _p(view.cols), view.n_rows, view.n_cols, m,
             warp_chunk, warps_per_cta, _p(w), _p(x), _p(y), f, nat.SCALING_CODES[scaling],
             _p(fin), _p(fout), _p(st_vals), _p(st_rows), dt, _p(ws),
             0 if ws is None else ws.numel(), _stream())
    Probe.launches += 2 + int(fin is not None)
    if staging:
        return y, st_rows[:nc], st_vals[:nc]
    return y


def spmm_vertex_ref(dg: DeviceGraph, x, scaling="post", norm="none", staging=False):
    """Vertex-grouped SpMMv, bit-exact with halfsparse.kernels.spmm_vertex_grouped."""
    view = dg.fwd
    _require_cuda(x)
    x = x.contiguous()
    f = x.shape[1]
    dt = _dtype_code(x)
    fin, fout = dg.norm_tables(norm, False, x.dtype)
    y = torch.empty((view.n_rows, f), dtype=x.dtype, device=x.device)
    gbase = st_rows = st_vals = None
    total = 0
    if staging:
        deg = view.offsets[1:] - view.offsets[:-1]
        ng = (deg + 31) // 32
        ng = torch.where(ng > 1, ng, torch.zeros_like(ng))
        csum = torch.cumsum(ng, 0)
        total = int(csum[-1].item()) if csum.numel() else 0
        gbase = (csum - ng).contiguous()
        st_rows = torch.empty(max(total, 1), dtype=torch.int64, device=x.device)
        st_vals = torch.empty((max(total, 1), f), dtype=x.dtype, device=x.device)
    ws = workspace(nat.size_query("hg_spmm_vertex_ref_workspace", view.n_cols, f,
                                  int(fin is not None), dt), x.device)
    nat.call("hg_spmm_vertex_ref", _p(view.offsets), _p(view.cols), view.n_rows, view.n_cols,
             _p(x), _p(y), f, nat.SCALING_CODES[scaling], _p(fin), _p(fout), _p(gbase),
             _p(st_vals), _p(st_rows), dt, _p(ws), 0 if ws is None else ws.numel(), _stream())
    if staging:
        return y, st_rows[:total], st_vals[:total]
    return y


# ── SDDMM, attention, softmax ────────────────────────────────────────────


def _butterfly_layout(x, y, f, heads):
    """Layouts hg_sddmm_fast runs on its butterfly kernels (and accepts packs
    for): F / V <= 32 with power-of-two head widths in V-element vectors."""
    fh = f // heads
    aligned = x.data_ptr() % 16 == 0 and y.data_ptr() % 16 == 0
    if x.dtype == torch.float16:
        v = 8 if aligned and fh % 8 == 0 else 2
    else:
        v = 4 if aligned and fh % 4 == 0 else 2
    g = fh // v
    return f // v <= 32 and g >= 1 and g & (g - 1) == 0 and (f // v) % g == 0


LANE32 = os.environ.get("HG_SPMM_LANE32", "1") != "0"


def _sddmm_lane32(x, y, f, heads):
    """hg_sddmm_fast's 32-byte-lane rule (binary16, 64..512 features, heads of
    16-element multiples, 32-byte aligned operands)."""
    return (LANE32 and x.dtype == torch.float16 and x.data_ptr() % 32 == 0
            and y.data_ptr() % 32 == 0 and (f // heads) % 16 == 0 and 64 <= f <= 512)


def sddmm(dg: DeviceGraph, x, y, heads=1, transpose=False, fast=False):
    """Per-edge (per-head) tree dot products, bit-exact with kernels.sddmm
    (fast=True: fp32 accumulation, one rounding -- hg_sddmm_fast).
    Returns [E] for heads == 1, else [E, heads]."""
    view = dg.view(transpose)
    _require_cuda(x, y)
    x, y = x.contiguous(), y.contiguous()
    if x.dtype != y.dtype:
        raise ValueError("operand modes differ")
    if x.shape[1] != y.shape[1]:
        raise ValueError("operand feature lengths differ")
    f = x.shape[1]
    out = torch.empty((view.num_edges, heads), dtype=x.dtype, device=x.device)
    if fast:
        # packs only for the 16-byte-lane kernels: with 32-byte lanes the unit
        # kernel alone was faster on RMAT-24 (F=128: 11.56 vs 11.78 ms)
        packed = (PACKING and view.n_rows >= PACK_MIN_ROWS and _butterfly_layout(x, y, f, heads)
                  and not _sddmm_lane32(x, y, f, heads))
        sched = view.schedule(DEFAULT_SPLIT_CAP, PACK_EDGES_WIDE if packed else -1)
        nat.call("hg_sddmm_fast", _p(view.offsets), _p(view.cols), view.n_rows, view.num_edges,
                 _p(sched.units), sched.num_units, _p(sched.packs), sched.num_packs,
                 _p(view.row_ids() if sched.num_packs else None), _p(x), _p(y), _p(out), f,
                 heads, _dtype_code(x), _stream())
        Probe.launches += 1 + int(sched.num_packs > 0)
    else:
        sched = view.schedule()
        nat.call("hg_sddmm", _p(view.offsets), _p(view.cols), view.n_rows, view.num_edges,
                 _p(sched.units), sched.num_units, _p(x), _p(y), _p(out), f, heads,
                 _dtype_code(x), _stream())
        Probe.launches += 1
    return out[:, 0] if heads == 1 else out


def attention_logits(dg: DeviceGraph, s_l, s_r, slope=0.2):
    """leaky_relu(attention_scores(s_l, s_r)) per head: [E, H]."""
    _require_cuda(s_l, s_r)
    s_l, s_r = s_l.contiguous(), s_r.contiguous()
    heads = s_l.shape[1] if s_l.dim() == 2 else 1
    out = torch.empty((dg.num_edges, heads), dtype=s_l.dtype, device=s_l.device)
    nat.call("hg_attn_scores", _p(dg.offsets), _p(dg.cols), dg.n, dg.num_edges, _p(s_l),
             _p(s_r), heads, float(slope), _p(out), _dtype_code(s_l), _stream())
    Probe.launches += 1
    return out


def softmax_fwd_view(view: CsrView, e):
    _require_cuda(e)
    e = e.contiguous()
    heads = e.shape[1] if e.dim() == 2 else 1
    alpha = torch.empty_like(e)
    lr = view.long_rows()
    nat.call("hg_edge_softmax_fwd", _p(view.offsets), view.n_rows, view.num_edges, _p(e),
             _p(alpha), heads, _p(lr), lr.numel(), LONG_ROW, _dtype_code(e), _stream())
    Probe.launches += 1 + int(lr.numel() > 0)
    return alpha


def softmax_bwd_view(view: CsrView, alpha, g):
    alpha, g = alpha.contiguous(), g.contiguous()
    heads = alpha.shape[1] if alpha.dim() == 2 else 1
    de = torch.empty_like(alpha)
    lr = view.long_rows()
    nat.call("hg_edge_softmax_bwd", _p(view.offsets), view.n_rows, view.num_edges, _p(alpha),
             _p(g), _p(de), heads, _p(lr), lr.numel(), LONG_ROW, _dtype_code(alpha), _stream())
    Probe.launches += 1 + int(lr.numel() > 0)
    return de


def rowsum_view(view: CsrView, v, perm=None):
    v = v.contiguous()
    heads = v.shape[1] if v.dim() == 2 else 1
    out = torch.empty((view.n_rows, heads), dtype=v.dtype, device=v.device)
    lr = view.long_rows()
    nat.call("hg_edge_rowsum", _p(view.offsets), view.n_rows, view.num_edges, _p(v), _p(perm),
             heads, _p(out), _p(lr), lr.numel(), LONG_ROW, _dtype_code(v), _stream())
    Probe.launches += 1 + int(lr.numel() > 0)
    return out


def _heads_of(s):
    return s.shape[1] if s.dim() == 2 else 1


def gat_attention_fwd(view: CsrView, s_l, s_r, slope=0.2, out=None):
    """Fused fp32-guarded leaky(s_l[r] + s_r[c]) -> edge softmax: alpha [E, H]
    (out: an [E, H] view with unit column stride, e.g. the alpha half of
    interleaved [E, 2H] rows)."""
    _require_cuda(s_l, s_r)
    s_l, s_r = s_l.contiguous(), s_r.contiguous()
    h = _heads_of(s_l)
    alpha = out if out is not None else torch.empty((view.num_edges, h), dtype=s_l.dtype,
                                                    device=s_l.device)
    med, lng = view.row_classes()
    nat.call("hg_gat_attention_fwd", _p(view.offsets), _p(view.cols), view.n_rows, _p(s_l),
             _p(s_r), h, float(slope), _p(alpha), alpha.stride(0), _p(med), med.numel(), _p(lng),
             lng.numel(), SHORT_ROW, _dtype_code(s_l), _stream())
    Probe.launches += 1
    return alpha


def gat_attention_stats(view: CsrView, s_l, s_r, slope=0.2):
    """Per-row softmax statistics of leaky(s_l[r] + s_r[c]): float32 [N, H, 2]
    = (log2-domain max, 1 / exp-sum) (hg_gat_attention_stats)."""
    _require_cuda(s_l, s_r)
    s_l, s_r = s_l.contiguous(), s_r.contiguous()
    h = _heads_of(s_l)
    stats = torch.empty((view.n_rows, h, 2), dtype=torch.float32, device=s_l.device)
    med, lng = view.row_classes()
    nat.call("hg_gat_attention_stats", _p(view.offsets), _p(view.cols), view.n_rows, _p(s_l),
             _p(s_r), h, float(slope), _p(stats), _p(med), med.numel(), _p(lng), lng.numel(),
             SHORT_ROW, _dtype_code(s_l), _stream())
    Probe.launches += 1
    return stats


def gat_aggregate(view: CsrView, z, s_l, s_r, stats, heads, slope=0.2, relu=False,
                  split_cap: int = DEFAULT_SPLIT_CAP):
    """Fused GAT forward core: (y [N, F], alpha [E, H]) with y[r] = sum_e alpha_e
    z[c_e] per head and alpha formed in the gather loop from s_l, s_r and
    `stats` (hg_gat_aggregate) -- bitwise equal to gat_attention_fwd followed
    by spmm_csr(view, z, alpha, heads=heads) on the same schedule."""
    _require_cuda(z, s_l, s_r, stats)
    z = z.contiguous()
    s_l, s_r = s_l.contiguous(), s_r.contiguous()
    if z.dim() != 2 or z.shape[0] != view.n_cols:
        raise ValueError(f"feature tensor has {z.shape[0]} rows for {view.n_cols} columns")
    f = z.shape[1]
    dt = _dtype_code(z)
    pack_edges = -1
    if PACKING and view.n_rows >= PACK_MIN_ROWS:
        pack_edges = PACK_EDGES_WIDE if f * z.element_size() >= 256 else PACK_EDGES_NARROW
    sched = view.schedule(split_cap, pack_edges)
    out = torch.empty((view.n_rows, f), dtype=z.dtype, device=z.device)
    alpha = torch.empty((view.num_edges, heads), dtype=z.dtype, device=z.device)
    nbytes = nat.size_query("hg_spmm_workspace", view.n_cols, f, sched.num_slots, 0, 0, dt)
    ws = workspace(nbytes, z.device)
    if Probe.timing:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    nat.call("hg_gat_aggregate", _p(view.offsets), _p(view.cols), view.n_rows, view.n_cols,
             view.num_edges, _p(sched.units), sched.num_units, _p(sched.split_rows),
             sched.split_rows.shape[0], sched.num_slots, _p(sched.packs), sched.num_packs,
             _p(view.row_ids() if sched.num_packs else None), _p(s_l), _p(s_r), _p(stats),
             float(slope), _p(alpha), heads, _p(z), _p(out), f, z.stride(0), out.stride(0),
             int(relu), dt, _p(ws), 0 if ws is None else ws.numel(), _stream())
    Probe.launches += int(sched.num_units > 0) + int(sched.num_packs > 0) + int(
        sched.split_rows.shape[0] > 0)
    if Probe.timing:
        ev1.record()
        Probe.records.append((ev0, ev1, spmm_bytes(view.n_rows, view.n_cols, view.num_edges, f,
                                                   heads, z.element_size()),
                              compulsory_bytes(view.n_rows, view.n_cols, view.num_edges, f,
                                               heads, z.element_size()),
                              (view.cols, view.num_edges, z, f) if Probe.keep else None,
                              (-(-f * z.element_size() // 16) * 16, view.num_edges)))
    return out, alpha


def gat_attention_bwd(view: CsrView, s_l, s_r, alpha, dalpha, slope=0.2, de_out=None):
    """(de [E, H], ds_l [N, H]) of gat_attention_fwd.  With de_out (the d_e half
    of interleaved [E, 2H] rows, alpha its other half) the two share one row
    stride."""
    s_l, s_r = s_l.contiguous(), s_r.contiguous()
    h = _heads_of(s_l)
    dalpha = dalpha.contiguous().view(alpha.shape[0], h)
    if de_out is None:
        alpha = alpha.contiguous()
        de = torch.empty_like(alpha)
    else:
        de = de_out
        if alpha.stride(0) != de.stride(0):
            raise ValueError("alpha and d_e must share a row stride")
    ds_l = torch.empty_like(s_l)
    med, lng = view.row_classes()
    nat.call("hg_gat_attention_bwd", _p(view.offsets), _p(view.cols), view.n_rows, _p(s_l),
             _p(s_r), h, float(slope), _p(alpha), _p(dalpha), _p(de), alpha.stride(0),
             _p(ds_l), _p(med), med.numel(), _p(lng), lng.numel(), SHORT_ROW,
             _dtype_code(s_l), _stream())
    Probe.launches += 1
    return de, ds_l


def edge_sums_fast(view: CsrView, v, perm=None):
    """out[r, h] = rnd(sum over row r of v[perm[e] or e, h]), fp32 accumulation."""
    v = v.contiguous()
    h = _heads_of(v)
    out = torch.empty((view.n_rows, h), dtype=v.dtype, device=v.device)
    med, lng = view.row_classes()
    nat.call("hg_edge_sums_fast", _p(view.offsets), view.n_rows, _p(v), _p(perm), h, _p(out),
             _p(med), med.numel(), _p(lng), lng.numel(), SHORT_ROW, _dtype_code(v), _stream())
    Probe.launches += 1
    return out


def head_mean(y, heads):
    """Mean over concatenated heads, fp64 sum, one rounding: [N, H*f] -> [N, f]."""
    y = y.contiguous()
    n, hf = y.shape
    out = torch.empty((n, hf // heads), dtype=y.dtype, device=y.device)
    nat.call("hg_head_mean", _p(y), n, heads, hf // heads, _p(out), _dtype_code(y), _stream())
    Probe.launches += 1
    return out


def head_mean_bwd(g, heads):
    g = g.contiguous()
    n, f = g.shape
    gin = torch.empty((n, heads * f), dtype=g.dtype, device=g.device)
    nat.call("hg_head_mean_bwd", _p(g), n, heads, f, _p(gin), _dtype_code(g), _stream())
    Probe.launches += 1
    return gin


def edge_softmax_fwd(dg: DeviceGraph, e):
    return softmax_fwd_view(dg.fwd, e)


def edge_softmax_bwd(dg: DeviceGraph, alpha, g):
    return softmax_bwd_view(dg.fwd, alpha, g)


def edge_rowsum(dg: DeviceGraph, v, transpose=False):
    """Per-row (transpose=False) or per-column (True) sums of per-edge values."""
    view = dg.view(transpose)
    return rowsum_view(view, v, view.perm if transpose else None)


def gemm_tc(a, bt, bias=None, row_scale=None, out=None, relu=False):
    """rnd(rnd(rnd(a @ bt.T) + bias) * row_scale[:, None]) (then max(., 0) with
    relu) on the tcgen05 tensor cores (hg_gemm_tc): a [M, K] fp16, bt [N, K]
    fp16 (N % 8 == 0)."""
    _require_cuda(a, bt)
    if a.dtype != torch.float16 or bt.dtype != torch.float16:
        raise ValueError("hg_gemm_tc takes binary16 operands")
    a, bt = a.contiguous(), bt.contiguous()
    if a.data_ptr() % 16:
        a = a.clone()
    if bt.data_ptr() % 16:
        bt = bt.clone()
    m, k = a.shape
    n, k2 = bt.shape
    if k2 != k:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float16, device=a.device)
    nat.call("hg_gemm_tc", _p(a), m, k, a.stride(0), _p(bt), n, bt.stride(0),
             _p(None if bias is None else bias.contiguous()),
             _p(None if row_scale is None else row_scale.contiguous()), int(relu), _p(out),
             out.stride(0), _stream())
    Probe.launches += 1
    return out


def gemm_tc_dots(a, bt, a_l, a_r, heads):
    """(z, s_l, s_r): z = rnd(a @ bt.T) on the tcgen05 tensor cores with the GAT
    head dots s_l[n, h] = rnd(sum_f z[n, h, f] a_l[h, f]) (s_r likewise, fp32
    sums of exact products of the rounded z) formed in the same epilogue
    (hg_gemm_tc_dots): N / heads a multiple of 16, heads <= 8."""
    _require_cuda(a, bt)
    if a.dtype != torch.float16 or bt.dtype != torch.float16:
        raise ValueError("hg_gemm_tc_dots takes binary16 operands")
    a, bt = a.contiguous(), bt.contiguous()
    if a.data_ptr() % 16:
        a = a.clone()
    if bt.data_ptr() % 16:
        bt = bt.clone()
    m, k = a.shape
    n, k2 = bt.shape
    if k2 != k:
        raise ValueError(f"inner dimensions differ: {k} vs {k2}")
    a_l = a_l.to(torch.float16).contiguous()
    a_r = a_r.to(torch.float16).contiguous()
    if a_l.numel() != n or a_r.numel() != n:
        raise ValueError("head vectors must hold heads x (N / heads) values")
    out = torch.empty((m, n), dtype=torch.float16, device=a.device)
    s_l = torch.empty((m, heads), dtype=torch.float16, device=a.device)
    s_r = torch.empty_like(s_l)
    nat.call("hg_gemm_tc_dots", _p(a), m, k, a.stride(0), _p(bt), n, bt.stride(0), _p(out),
             out.stride(0), _p(a_l), _p(a_r), heads, _p(s_l), _p(s_r), _stream())
    Probe.launches += 1
    return out, s_l, s_r


def gemm_tc_masked(a, bt, mask):
    """The ReLU backward folded into dX: y = rnd(a @ bt.T) where mask > 0,
    else +0 (relu_grad(mask, a @ bt.T), models.py:176-185) on the tcgen05
    tensor cores (hg_gemm_tc_masked): a [M, K], bt [N, K], mask [M, N] fp16,
    N a multiple of 16."""
    _require_cuda(a, bt)
    if a.dtype != torch.float16 or bt.dtype != torch.float16 or mask.dtype != torch.float16:
        raise ValueError("hg_gemm_tc_masked takes binary16 operands")
    a, bt = a.contiguous(), bt.contiguous()
    if a.data_ptr() % 16:
        a = a.clone()
    if bt.data_ptr() % 16:
        bt = bt.clone()
    m, k = a.shape
    n, k2 = bt.shape
    if k2 != k or mask.shape != (m, n):
        raise ValueError("shapes: a [M, K], bt [N, K], mask [M, N]")
    if mask.stride(1) != 1 or mask.stride(0) % 8 or mask.data_ptr() % 16:
        mask = mask.contiguous().clone()
    out = torch.empty((m, n), dtype=torch.float16, device=a.device)
    nat.call("hg_gemm_tc_masked", _p(a), m, k, a.stride(0), _p(bt), n, bt.stride(0), _p(out),
             out.stride(0), _p(mask), mask.stride(0), _stream())
    Probe.launches += 1
    return out


def gemm_wgrad(a, b, out=None, bias_out=None, accumulate=False, bias=False):
    """rnd(a.T @ b) -- fp32 accumulation, one rounding -- on the tcgen05 tensor
    cores with the vertex dimension split across the SMs (hg_gemm_wgrad):
    a [K, M] fp16 (layer input), b [K, N] fp16 (output gradient), M and N
    multiples of 8, N <= 256.  With bias (or a bias_out buffer) the column sums
    rnd(sum_k b[k, :]) come out of the same pass; returns (dW, db) then.  With
    accumulate, out = rnd(out + a.T @ b) (and likewise bias_out): autograd's
    gradient accumulation into a leaf, done in the kernel."""
    _require_cuda(a, b)
    if a.dtype != torch.float16 or b.dtype != torch.float16:
        raise ValueError("hg_gemm_wgrad takes binary16 operands")
    a, b = a.contiguous(), b.contiguous()
    if a.data_ptr() % 16:
        a = a.clone()
    if b.data_ptr() % 16:
        b = b.clone()
    k, m = a.shape
    k2, n = b.shape
    if k2 != k:
        raise ValueError(f"row counts differ: {k} vs {k2}")
    if accumulate and (out is None or ((bias or bias_out is not None) and bias_out is None)):
        raise ValueError("accumulate needs the output buffers")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float16, device=a.device)
    if bias and bias_out is None:
        bias_out = torch.empty(n, dtype=torch.float16, device=a.device)
    nbytes = nat.size_query("hg_gemm_wgrad_workspace", k, m, n)
    ws = workspace(nbytes, a.device)
    nat.call("hg_gemm_wgrad", _p(a), k, m, a.stride(0), _p(b), n, b.stride(0), _p(out),
             out.stride(0), _p(bias_out), int(accumulate), _p(ws),
             0 if ws is None else ws.numel(), _stream())
    Probe.launches += 2 if k else 1
    return out if bias_out is None else (out, bias_out)


def bias_scale_rows(x, bias=None, row_scale=None, out=None):
    """rnd(rnd(x + bias[None, :]) * row_scale[:, None]) (hg_bias_scale_rows);
    either operand may be None."""
    _require_cuda(x)
    x = x.contiguous()
    rows, f = x.shape
    for t in (bias, row_scale):
        if t is not None and t.dtype != x.dtype:
            raise ValueError("bias / row scale must match the feature dtype")
    if out is None:
        out = torch.empty_like(x)
    nat.call("hg_bias_scale_rows", _p(x), _p(None if bias is None else bias.contiguous()),
             _p(None if row_scale is None else row_scale.contiguous()), rows, f, _p(out),
             _dtype_code(x), _stream())
    Probe.launches += 1
    return out


def scale_combine(x, a, one_plus_eps, lam):
    """GIN combine rnd(rnd(x * ope) + rnd(a * lam)) in one pass (hg_scale_combine)."""
    _require_cuda(x, a)
    x, a = x.contiguous(), a.contiguous()
    out = torch.empty_like(x)
    nat.call("hg_scale_combine", _p(x), _p(a), _p(one_plus_eps.contiguous()), float(lam),
             x.numel(), _p(out), _dtype_code(x), _stream())
    Probe.launches += 1
    return out


def scale_combine_bwd(x, g, one_plus_eps, lam, need_gx=True, need_ga=True, need_gope=True):
    """(gx, ga, gope) of scale_combine; entries not needed are None."""
    g = g.contiguous()
    x = x.contiguous()
    gx = torch.empty_like(g) if need_gx else None
    ga = torch.empty_like(g) if need_ga else None
    gope = torch.empty_like(one_plus_eps) if need_gope else None
    ws = workspace(nat.size_query("hg_scale_combine_bwd_workspace"), g.device) if need_gope else None
    nat.call("hg_scale_combine_bwd", _p(x), _p(g), _p(one_plus_eps.contiguous()), float(lam),
             g.numel(), _p(gx), _p(ga), _p(gope), _dtype_code(g), _p(ws),
             0 if ws is None else ws.numel(), _stream())
    Probe.launches += 1 + int(need_gope)
    return gx, ga, gope


def gather_rows(src, idx):
    """src[idx] along dim 0 (int32 idx), one pass (hg_gather_rows)."""
    src = src.contiguous()
    rows = idx.numel()
    out = torch.empty((rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 0
    if rows and row_bytes:
        nat.call("hg_gather_rows", _p(src), _p(idx), rows, row_bytes, _p(out), _stream())
        Probe.launches += 1
    return out


def relu_grad(y, g):
    """g where y > 0 else 0 (y = the ReLU's output), one pass (hg_relu_grad)."""
    y, g = y.contiguous(), g.contiguous()
    out = torch.empty_like(g)
    nat.call("hg_relu_grad", _p(y), _p(g), g.numel(), _p(out), _dtype_code(g), _stream())
    Probe.launches += 1
    return out


def col_sums(x):
    """rnd(sum over rows) per column, fp32 accumulation (hg_col_sums)."""
    _require_cuda(x)
    x = x.contiguous()
    rows, f = x.shape
    out = torch.empty(f, dtype=x.dtype, device=x.device)
    nbytes = nat.size_query("hg_col_sums_workspace", rows, f)
    ws = workspace(nbytes, x.device)
    nat.call("hg_col_sums", _p(x), rows, f, _p(out), _dtype_code(x), _p(ws), ws.numel(),
             _stream())
    Probe.launches += 2
    return out


def scale_f64(x, s: float):
    """rnd(x * s) with the product formed in float64."""
    x = x.contiguous()
    out = torch.empty_like(x)
    nat.call("hg_scale_f64", _p(x), float(s), _p(out), x.numel(), _dtype_code(x), _stream())
    Probe.launches += 1
    return out


def softmax_xent(logits, labels, c_active, denom, scale=1.0, grad_dtype=None):
    """Fused fp64 softmax cross-entropy on fp16 or fp32 logits: returns
    (nll [N] f64, grad [N, ld] of grad_dtype (default the logits' dtype)),
    grad = rnd(fp32((p - y) / denom) * scale)."""
    logits = logits.contiguous()
    n, ld = logits.shape
    grad = torch.empty((n, ld), dtype=grad_dtype or logits.dtype, device=logits.device)
    nll = torch.empty(n, dtype=torch.float64, device=logits.device)
    nat.call("hg_softmax_xent", _p(logits), _dtype_code(logits), ld, _p(labels), n, c_active,
             float(denom), float(scale), _p(grad), _dtype_code(grad), _p(nll), _stream())
    Probe.launches += 1
    return nll, grad


def head_dots(z, a_l, a_r, heads):
    """s_l[n, h] = z[n, h, :] . a_l[h, :], s_r likewise (fp32 accumulate, one rounding)."""
    z = z.contiguous()
    n = z.shape[0]
    fh = z.shape[1] // heads
    s_l = torch.empty((n, heads), dtype=z.dtype, device=z.device)
    s_r = torch.empty_like(s_l)
    nat.call("hg_head_dots", _p(z), _p(a_l.contiguous()), _p(a_r.contiguous()), n, heads, fh,
             _p(s_l), _p(s_r), _dtype_code(z), _stream())
    Probe.launches += 1
    return s_l, s_r


def adam_step(master, m, v, grad, lr, b1, b2, eps, step, grad_unscale=1.0, pub=None,
              grad_zero=None, step_done=None, transposed=None, pub_t=None):
    """One fused Adam update over flat fp32 arrays (hg_adam_step); `step` is the
    device fp64 step count (already incremented -- or, with step_done (an int32
    zero counter), advanced by the kernel itself); the gradient is multiplied
    by grad_unscale (exact for a power of two) before use.  pub: also write the
    next step's published copy rnd(master); transposed [(offset, K, N,
    offset_in_pub_t)] + pub_t: and the transposed copies of those 2-D weights;
    grad_zero: a gradient buffer of pub's dtype to clear for the next step."""
    pdt = _dtype_code(pub if pub is not None else (grad_zero if grad_zero is not None else grad))
    tl = list(transposed or []) if pub_t is not None else []
    desc = (ctypes.c_int64 * max(1, 4 * len(tl)))(*[int(v) for t in tl for v in t])
    nat.call("hg_adam_step", _p(master), _p(m), _p(v), _p(grad), _dtype_code(grad),
             master.numel(), float(lr), float(1 - b1), float(1 - b2), float(b1), float(b2),
             float(eps), _p(step), float(grad_unscale), _p(pub), _p(grad_zero), pdt,
             _p(step_done), desc, len(tl), _p(pub_t if tl else None), _stream())


_LOSS_WS = {}


def loss_mean(nll, denom):
    """fp32(sum(nll) / denom) as a device scalar (hg_loss_mean, fixed-order fp64
    sums; a dedicated zero-initialised scratch per (device, stream) holds the
    block partials and the arrival counter the kernel re-arms)."""
    key = (nll.device, torch.cuda.current_stream(nll.device).cuda_stream)
    ws = _LOSS_WS.get(key)
    if ws is None:
        ws = torch.zeros(nat.size_query("hg_loss_mean_workspace"), dtype=torch.uint8,
                         device=nll.device)
        _LOSS_WS[key] = ws
    out = torch.empty((), dtype=torch.float32, device=nll.device)
    nat.call("hg_loss_mean", _p(nll.contiguous()), nll.numel(), float(denom), _p(out), _p(ws),
             ws.numel(), _stream())
    Probe.launches += 1
    return out
    Probe.launches += 1


def head_dots_bwd(z, a_l, a_r, g_l, g_r, heads, gz_acc=None, dz=True):
    """Backward of head_dots: (gz, ga_l, ga_r), deterministic (hg_head_dots_bwd).
    gz_acc: an existing gradient of z to accumulate into (in place); dz=False:
    only (None, ga_l, ga_r) -- the dz term went into an aggregation's store."""
    z = z.contiguous()
    n = z.shape[0]
    fh = z.shape[1] // heads
    if not dz:
        gz = gz_acc = None
    else:
        gz = torch.empty_like(z) if gz_acc is None else gz_acc
    ga_l = torch.empty_like(a_l)
    ga_r = torch.empty_like(a_r)
    ws = workspace(nat.size_query("hg_head_dots_bwd_workspace", heads, fh), z.device)
    nat.call("hg_head_dots_bwd", _p(z), _p(a_l.contiguous()), _p(a_r.contiguous()),
             _p(g_l.contiguous()), _p(g_r.contiguous()), n, heads, fh, _p(gz), _p(ga_l),
             _p(ga_r), _p(gz_acc), _dtype_code(z), _p(ws), ws.numel(), _stream())
    Probe.launches += 2
    return gz, ga_l, ga_r


# ── multi-GPU exchange through the C ABI (callers with their own NCCL comm) ──


class NcclComm:
    """An NCCL communicator owned through the C ABI (hg_nccl_comm_init) -- the
    path a non-Python host uses for the row-partitioned exchange.  Rank 0
    makes the id (`unique_id()`) and shares it out of band."""

    def __init__(self, nranks: int, rank: int, uid: bytes):
        if len(uid) != 128:
            raise ValueError("an ncclUniqueId is 128 bytes")
        self.nranks, self.rank = nranks, rank
        self._uid = ctypes.create_string_buffer(uid, 128)
        self.handle = ctypes.c_void_p()
        nat.call("hg_nccl_comm_init", ctypes.byref(self.handle), nranks, self._uid, rank)

    @staticmethod
    def available() -> bool:
        return bool(nat.lib().hg_nccl_available())

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        nat.call("hg_nccl_unique_id", buf)
        return buf.raw

    def close(self):
        if self.handle:
            nat.call("hg_nccl_comm_destroy", self.handle)
            self.handle = ctypes.c_void_p()


def allgather_features(comm: NcclComm, x_local: torch.Tensor, splits, out=None):
    """hg_allgather_features: [N, ...] rows in global order from every rank's
    x_local (rows [splits[q], splits[q+1]) of rank q), exact counts."""
    _require_cuda(x_local)
    x_local = x_local.contiguous()
    sp = [int(v) for v in splits]
    n = sp[-1]
    tail = tuple(x_local.shape[1:])
    if out is None:
        out = x_local.new_empty((n,) + tail)
    row = x_local.element_size()
    for d in tail:
        row *= int(d)
    arr = (ctypes.c_int64 * len(sp))(*sp)
    nat.call("hg_allgather_features", comm.handle, _p(x_local), _p(out), arr, len(sp) - 1,
             comm.rank, row, _stream())
    return out

"""Tensor-level API over libixgpu.so.

Every function takes CUDA tensors (torch is used only for device memory and
streams) and calls exactly one C-ABI entry point on the current stream.
Data-dependent scalars come back as device tensors; nothing here
synchronises the host unless the caller reads a result.  There is no CPU
path: without libixgpu.so and an sm_100 device, the first call raises.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib as L
from .pred import Pred

_DT = {torch.int32: L.I32, torch.int64: L.I64, torch.uint8: L.U8, torch.bool: L.U8, torch.float64: L.F64}


def _lib():
    return L.load(require_device=True)


def _ptr(t: Optional[torch.Tensor]):
    """a tensor's device address for a void* argument (plain int: ctypes
    converts it without a wrapper object)"""
    return t.data_ptr() if t is not None and t.numel() > 0 else None


_raw_stream = torch._C._cuda_getCurrentRawStream


def _stream():
    """the current CUDA stream as a void* (the cheap raw query: a launch-bound
    call such as C1's 2^20 partition2 spends its time here otherwise)"""
    return _raw_stream(torch.cuda.current_device())


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}") from None


_PRED_CACHE: dict = {}


def _c_pred(p: Pred) -> L.ixg_pred:
    if not isinstance(p, Pred):
        raise TypeError(
            "predicate arguments must be paper_2506_23058_b200.Pred descriptors "
            f"(got {type(p).__name__}); opaque Python callables cannot run on the device"
        )
    key = (p.kind, p.thr, p.seed)
    c = _PRED_CACHE.get(key)
    if c is None:
        if len(_PRED_CACHE) > 1024:
            _PRED_CACHE.clear()
        c = _PRED_CACHE[key] = L.ixg_pred(p.kind, 0, p.thr, p.seed & ((1 << 64) - 1))
    return c


def _contig(t: torch.Tensor) -> torch.Tensor:
    t = t.contiguous()
    if t.numel() and t.data_ptr() % 16:
        t = t.clone()
    return t


# ------------------------------------------------------------------ workspace
class Workspace:
    """Per-(device, op, stream) scratch, zeroed whenever its layout (op, n, m)
    changes.  One workspace per stream: two streams running the same op never
    share look-back slots or tile tickets (one stream /
    workspace per concurrent caller).

    The kernels leave their look-back state ready for the next launch
    (epoch-tagged flags), so steady-state calls do no memset."""

    def __init__(self):
        self._bufs: dict = {}
        self._need: dict = {}

    def get(self, op: int, n: int, m: int, device) -> torch.Tensor:
        need = self._need.get((op, n, m))
        if need is None:
            if len(self._need) > 4096:
                self._need.clear()
            need = self._need[(op, n, m)] = int(_lib().ixg_ws_bytes(op, n, m))
        dev = device.index if isinstance(device, torch.device) else device
        if dev is None:
            dev = torch.cuda.current_device()
        key = (dev, op, _raw_stream(dev))
        ent = self._bufs.get(key)
        if ent is None or ent[1].numel() < need:
            buf = torch.zeros(max(need, 4096), dtype=torch.uint8, device=device)
            self._bufs[key] = ((n, m), buf)
            return buf
        if ent[0] != (n, m):
            ent[1].zero_()
            self._bufs[key] = ((n, m), ent[1])
        return ent[1]


WS = Workspace()


def _ws(op: int, n: int, m: int, device):
    buf = WS.get(op, n, m, device)
    return buf.data_ptr(), buf.numel()


# ------------------------------------------------------------------ status
@dataclass
class StatusView:
    first: int
    codes: int
    flags: int

    @property
    def ok(self) -> bool:
        return self.codes == 0

    @property
    def stmt(self) -> int:
        return (self.first >> 56) & 0xFF

    @property
    def elem(self) -> int:
        return (self.first >> 8) & 0xFFFFFFFFFFFF

    @property
    def site(self) -> int:
        return self.first & 0xFF

    @property
    def narrow(self) -> bool:
        return bool(self.flags & L.F_NARROW)


class Status:
    """Device-resident ixg_status (first failure in sequential order)."""

    def __init__(self, device=None):
        self.t = torch.empty(2, dtype=torch.int64, device=device or torch.device("cuda"))
        self.reset()

    def reset(self):
        L.check(_lib().ixg_status_init(_ptr(self.t), _stream()), "ixg_status_init")

    @property
    def ptr(self):
        return _ptr(self.t)

    def read(self) -> StatusView:
        h = self.t.cpu().numpy().view("uint64")
        return StatusView(int(h[0]), int(h[1]) & 0xFFFFFFFF, int(h[1]) >> 32)

    def read_with(self, *scalars: torch.Tensor):
        """The status and some device int64 scalars (counts) in one host
        round trip: async copies into a pinned buffer, one stream sync."""
        n = 2 + sum(int(t.numel()) for t in scalars)
        h = torch.empty(n, dtype=torch.int64, pin_memory=True)
        h[:2].copy_(self.t, non_blocking=True)
        o = 2
        for t in scalars:
            h[o:o + t.numel()].copy_(t.reshape(-1).to(torch.int64), non_blocking=True)
            o += t.numel()
        torch.cuda.current_stream(self.t.device).synchronize()
        u = h[:2].numpy().view("uint64")
        return StatusView(int(u[0]), int(u[1]) & 0xFFFFFFFF, int(u[1]) >> 32), h[2:].tolist()


# ------------------------------------------------------------------ builtins
def scan_add(xs: torch.Tensor, ne: int = 0, exclusive: bool = False, out=None, status=None) -> torch.Tensor:
    """scan (+) ne xs (oracle.py:281-293): int64 inclusive (or exclusive)
    sums; with a Status, the first sum that leaves int64 is recorded
    (IXG_OVERFLOW at site L.OVF_SITE)."""
    xs = _contig(xs)
    n = xs.numel()
    out = torch.empty(n, dtype=torch.int64, device=xs.device) if out is None else out
    ws, wsb = _ws(L.OP_SCAN, n, 0, xs.device)
    st = status.ptr if status is not None else _ptr(None)
    L.check(_lib().ixg_scan_add(_dt(xs), _ptr(xs), n, ne, int(exclusive), _ptr(out), ws, wsb, st, _stream()),
            "scan_add")
    return out


def reduce_add(xs: torch.Tensor, out=None) -> torch.Tensor:
    """total of scan (+) 0 xs (its last element) as a device int64 scalar."""
    xs = _contig(xs)
    out = torch.empty(1, dtype=torch.int64, device=xs.device) if out is None else out
    L.check(_lib().ixg_reduce_add(_dt(xs), _ptr(xs), xs.numel(), _ptr(out), _stream()), "reduce_add")
    return out


def jagged_dest(bits: torch.Tensor, cs: torch.Tensor, tb: torch.Tensor, out=None) -> torch.Tensor:
    """partition2L's scatter destinations (ixg_jagged_dest)."""
    cs, tb = _contig(cs), _contig(tb)
    n = cs.numel()
    out = torch.empty(n, dtype=torch.int64, device=cs.device) if out is None else out
    L.check(_lib().ixg_jagged_dest(_ptr(bits), n, _ptr(cs), _ptr(tb), _ptr(out), _stream()), "jagged_dest")
    return out


def segscan_add(flags: torch.Tensor, xs: torch.Tensor, want_flags: bool = False, status=None):
    """sgmSum's 2-ary scan; returns values (and flags).
    With a Status, a segment sum leaving int64 is recorded (L.OVF_SITE)."""
    flags, xs = _contig(flags), _contig(xs)
    n = flags.numel()
    out_v = torch.empty(n, dtype=torch.int64, device=xs.device)
    out_f = torch.empty(n, dtype=torch.uint8, device=xs.device) if want_flags else None
    ws, wsb = _ws(L.OP_SEGSCAN, n, 0, xs.device)
    st = status.ptr if status is not None else _ptr(None)
    L.check(
        _lib().ixg_segscan_add(_dt(flags), _ptr(flags), _dt(xs), _ptr(xs), n, 0, 0, _ptr(out_v), _ptr(out_f), ws, wsb,
                               st, _stream()),
        "segscan_add",
    )
    return (out_v, out_f) if want_flags else out_v


BIN_MIN_PAIRS = 1 << 22  # below this the destination is L2-sized anyway: direct


def scatter_layout(is_: torch.Tensor, ndst: int) -> int:
    """IXG_SCATTER_BINNED when `is_` has no locality (ixg_scatter_probe on
    the device; one 4-byte read back), else IXG_SCATTER_DIRECT."""
    if is_.numel() < BIN_MIN_PAIRS or not (1 << 23) < ndst <= (1 << 32):
        return L.SCATTER_DIRECT
    flag = torch.empty(1, dtype=torch.int32, device=is_.device)
    L.check(_lib().ixg_scatter_probe(_ptr(is_), is_.numel(), _ptr(flag), _stream()), "scatter_probe")
    return L.SCATTER_BINNED if int(flag.item()) else L.SCATTER_DIRECT


def scatter(out: torch.Tensor, is_: torch.Tensor, vs: torch.Tensor, site_bits: int, status: Status,
            stmt: int = 0, site: int = 0, layout="auto") -> torch.Tensor:
    """scatter into `out` in place (oracle.py:294-305); `out` already holds dst
    unless the site's V_INIT bit is clear.  layout: "auto" (probe the index
    array's locality), L.SCATTER_DIRECT or L.SCATTER_BINNED."""
    is_, vs = _contig(is_), _contig(vs)
    m = min(is_.numel(), vs.numel())
    if layout == "auto":
        layout = scatter_layout(is_[:m], out.numel())
    op = L.OP_SCATTER_BINNED if layout == L.SCATTER_BINNED else L.OP_SCATTER
    ws, wsb = _ws(op, m, out.numel(), out.device)
    L.check(
        _lib().ixg_scatter(_dt(out), _ptr(out), out.numel(), _ptr(is_), is_.numel(), _ptr(vs), vs.numel(),
                           site_bits, stmt, site, layout, status.ptr, ws, wsb, _stream()),
        "scatter",
    )
    return out


def gather(arr: torch.Tensor, idx: torch.Tensor, site_bits: int, status: Status, stmt: int = 0, site: int = 0):
    """out[i] = arr[idx[i]] with (V_BOUNDS) or without the bounds check."""
    arr, idx = _contig(arr), _contig(idx)
    out = torch.empty(idx.numel(), dtype=arr.dtype, device=idx.device)
    if arr.numel() == 0 and idx.numel() and not (site_bits & L.V_BOUNDS):
        raise ValueError("elided gather from an empty array")
    L.check(
        _lib().ixg_gather(_dt(arr), _ptr(arr), arr.numel(), _ptr(idx), idx.numel(), _ptr(out), site_bits, stmt, site,
                          status.ptr, _stream()),
        "gather",
    )
    return out


def hist(op: int, ne: int, dlen: int, is_: torch.Tensor, vs: torch.Tensor, status=None) -> torch.Tensor:
    """hist op ne dlen is vs (oracle.py:306-316).  (+) bins are summed in
    128 bits; with a Status, a bin whose sum leaves int64 is recorded."""
    is_, vs = _contig(is_), _contig(vs)
    out = torch.empty(max(dlen, 0), dtype=torch.int64, device=is_.device)
    ws, wsb = _ws(L.OP_HIST, 0, max(dlen, 0), is_.device) if op == L.HIST_ADD else (None, 0)
    st = status.ptr if status is not None else _ptr(None)
    L.check(
        _lib().ixg_hist(op, ne, dlen, _ptr(is_), is_.numel(), _ptr(vs), vs.numel(), _ptr(out), ws, wsb, st, _stream()),
        "hist"
    )
    return out


def fill(n: int, v: int, dtype=torch.int64, device=None) -> torch.Tensor:
    out = torch.empty(max(n, 0), dtype=dtype, device=device or torch.device("cuda"))
    L.check(_lib().ixg_fill(_dt(out), _ptr(out), out.numel(), int(v), _stream()), "fill")
    return out


def iota(n: int, device=None) -> torch.Tensor:
    out = torch.empty(max(n, 0), dtype=torch.int64, device=device or torch.device("cuda"))
    L.check(_lib().ixg_iota(_ptr(out), out.numel(), _stream()), "iota")
    return out


# ------------------------------------------------------------------ pipelines
def filter(xs: torch.Tensor, p: Pred, variant: int, status: Status, ys=None, d_count=None):
    """filter p xs (corpus filter.ixl); returns (ys capacity buffer, device count)."""
    xs = _contig(xs)
    n = xs.numel()
    ys = torch.empty(n, dtype=xs.dtype, device=xs.device) if ys is None else ys
    d_count = torch.empty(1, dtype=torch.int64, device=xs.device) if d_count is None else d_count
    ws, wsb = _ws(L.OP_FILTER, n, 0, xs.device)
    cp = _c_pred(p)
    L.check(
        _lib().ixg_filter(_dt(xs), _ptr(xs), n, ctypes.byref(cp), _ptr(ys), _ptr(d_count), variant, status.ptr, ws, wsb,
                          _stream()),
        "filter",
    )
    return ys, d_count


def filter_by(cs: torch.Tensor, xs: torch.Tensor, variant: int, status: Status):
    """filter_by cs xs (maxmatching.ixl:1-9)."""
    cs, xs = _contig(cs.view(torch.uint8) if cs.dtype == torch.bool else cs.to(torch.uint8)), _contig(xs)
    n = xs.numel()
    ys = torch.empty(n, dtype=xs.dtype, device=xs.device)
    d_count = torch.empty(1, dtype=torch.int64, device=xs.device)
    ws, wsb = _ws(L.OP_FILTER, n, 0, xs.device)
    L.check(
        _lib().ixg_filter_by(_dt(xs), _ptr(cs), _ptr(xs), n, _ptr(ys), _ptr(d_count), variant, status.ptr, ws, wsb,
                             _stream()),
        "filter_by",
    )
    return ys, d_count


def partition2(xs: torch.Tensor, p: Pred, variant: int, status: Status, ys=None, d_nt=None):
    """partition2 p xs (corpus partition2.ixl); returns (ys, device num_true)."""
    xs = _contig(xs)
    n = xs.numel()
    ys = torch.empty(n, dtype=xs.dtype, device=xs.device) if ys is None else ys
    d_nt = torch.empty(1, dtype=torch.int64, device=xs.device) if d_nt is None else d_nt
    ws, wsb = _ws(L.OP_PARTITION2, n, 0, xs.device)
    cp = _c_pred(p)
    L.check(
        _lib().ixg_partition2(_dt(xs), _ptr(xs), n, ctypes.byref(cp), _ptr(ys), _ptr(d_nt), variant, status.ptr, ws,
                              wsb, _stream()),
        "partition2",
    )
    return ys, d_nt


def partition_counts(xs: torch.Tensor, p: Pred, q: Optional[Pred] = None, d_tot=None) -> torch.Tensor:
    """class totals of xs for partition2 (q None: [trues]) or partition3
    ([class 0, class 1]) as a device int64 tensor."""
    xs = _contig(xs)
    classes = 2 if q is None else 3
    d_tot = torch.empty(classes - 1, dtype=torch.int64, device=xs.device) if d_tot is None else d_tot
    ws, wsb = _ws(L.OP_PARTITION2, xs.numel(), 0, xs.device)
    cp = _c_pred(p)
    cq = _c_pred(q) if q is not None else None
    L.check(_lib().ixg_partition_counts(_dt(xs), _ptr(xs), xs.numel(), ctypes.byref(cp),
                                        ctypes.byref(cq) if cq is not None else None, classes, _ptr(d_tot), ws, wsb,
                                        _stream()), "partition_counts")
    return d_tot


def partition2_peer(xs: torch.Tensor, p: Pred, dst_ptrs, shard: int, d_counts: torch.Tensor, rank: int) -> None:
    """this rank's partition2 runs stored straight into the sharded global
    output (dst_ptrs[r] = rank r's shard, peer-mapped; d_counts = every
    rank's true count on the device; see ixg_partition2_peer)."""
    xs = _contig(xs)
    n = xs.numel()
    ws, wsb = _ws(L.OP_PARTITION2, n, 0, xs.device)
    cp = _c_pred(p)
    arr = (ctypes.c_void_p * len(dst_ptrs))(*[int(x) for x in dst_ptrs])
    L.check(_lib().ixg_partition2_peer(_dt(xs), _ptr(xs), n, ctypes.byref(cp), arr, len(dst_ptrs), shard,
                                       _ptr(d_counts), rank, ws, wsb, _stream()), "partition2_peer")


def rank_offsets(d_counts: torch.Tensor, ranks: int, rank: int, stride: int = 1, out=None) -> torch.Tensor:
    """[this rank's exclusive offset, the total] of an all-gathered device
    count array (ixg_rank_offsets)."""
    out = torch.empty(2, dtype=torch.int64, device=d_counts.device) if out is None else out
    L.check(_lib().ixg_rank_offsets(_ptr(d_counts), ranks, rank, stride, _ptr(out), _stream()), "rank_offsets")
    return out


class DeviceBuffer:
    """cudaMalloc'd buffer (exactly its own IPC allocation) viewed as a tensor."""

    def __init__(self, n: int, dtype=torch.int32, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.nbytes = n * torch.empty(0, dtype=dtype).element_size()
        ptr = ctypes.c_void_p()
        L.check(_lib().ixg_dev_alloc(self.nbytes, ctypes.byref(ptr)), "dev_alloc")
        self.ptr = ptr.value
        typestr = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (self.ptr, False), "version": 2}

        self.tensor = torch.as_tensor(_View(), device=dev)

    def ipc_handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        L.check(_lib().ixg_ipc_handle(self.ptr, h), "ipc_handle")
        return h.raw

    def free(self):
        if self.ptr:
            L.check(_lib().ixg_dev_free(self.ptr), "dev_free")
            self.ptr = None


def ipc_open(handle: bytes) -> int:
    ptr = ctypes.c_void_p()
    L.check(_lib().ixg_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)), "ipc_open")
    return ptr.value


def ipc_close(ptr: int) -> None:
    L.check(_lib().ixg_ipc_close(ptr), "ipc_close")


def partition3(xs: torch.Tensor, p: Pred, q: Pred, variant: int, status: Status, ys=None, d_m=None):
    """partition3 p q xs (corpus partition3.ixl); returns (ys, device (m1, m2))."""
    xs = _contig(xs)
    n = xs.numel()
    ys = torch.empty(n, dtype=xs.dtype, device=xs.device) if ys is None else ys
    d_m = torch.empty(2, dtype=torch.int64, device=xs.device) if d_m is None else d_m
    ws, wsb = _ws(L.OP_PARTITION3, n, 0, xs.device)
    cp, cq = _c_pred(p), _c_pred(q)
    L.check(
        _lib().ixg_partition3(_dt(xs), _ptr(xs), n, ctypes.byref(cp), ctypes.byref(cq), _ptr(ys), _ptr(d_m), variant,
                              status.ptr, ws, wsb, _stream()),
        "partition3",
    )
    return ys, d_m


def c2(xs: torch.Tensor, p: Pred, shape: torch.Tensor, variant: int, status: Status, z_dtype=None, ys=None, zs=None,
       d_k=None):
    """c2 p xs shape = filter + mkFlags + sgmSum (corpus/c2_filter_sgmsum.ixl)."""
    xs, shape = _contig(xs), _contig(shape.to(torch.int64))
    n, m = xs.numel(), shape.numel()
    z_dtype = z_dtype or xs.dtype
    ys = torch.empty(n, dtype=xs.dtype, device=xs.device) if ys is None else ys
    zs = torch.empty(n, dtype=z_dtype, device=xs.device) if zs is None else zs
    d_k = torch.empty(1, dtype=torch.int64, device=xs.device) if d_k is None else d_k
    ws, wsb = _ws(L.OP_C2, n, m, xs.device)
    cp = _c_pred(p)
    L.check(
        _lib().ixg_c2(_dt(xs), _ptr(xs), n, ctypes.byref(cp), _ptr(shape), m, _ptr(ys), _dt(zs), _ptr(zs), _ptr(d_k),
                      variant, status.ptr, ws, wsb, _stream()),
        "c2",
    )
    return ys, zs, d_k


def mksgmdescr(shape: torch.Tensor, xs: torch.Tensor, variant: int, status: Status):
    """mkSgmDescr shape xs (corpus mksgmdescr.ixl).  Two calls: the first
    computes len = sum shape on the device, the second scatters into
    `replicate len 0` (the result length is data-dependent)."""
    shape, xs = _contig(shape), _contig(xs)
    m = shape.numel()
    d_len = torch.empty(1, dtype=torch.int64, device=xs.device)
    ws, wsb = _ws(L.OP_MKSGMDESCR, 0, m, xs.device)
    lib = _lib()
    L.check(lib.ixg_mksgmdescr(_ptr(shape), _ptr(xs), m, xs.numel(), _ptr(None), 0, _ptr(d_len), variant, status.ptr,
                               ws, wsb, _stream()), "mksgmdescr")
    cap = int(d_len.item())
    res = torch.empty(max(cap, 0), dtype=torch.int64, device=xs.device)
    if cap > 0:
        ws, wsb = _ws(L.OP_MKSGMDESCR, cap, m, xs.device)
        L.check(lib.ixg_mksgmdescr(_ptr(shape), _ptr(xs), m, xs.numel(), _ptr(res), cap, _ptr(d_len), variant,
                                   status.ptr, ws, wsb, _stream()), "mksgmdescr")
    return res


def mkflags(k: int, shape: torch.Tensor, variant: int, status: Status) -> torch.Tensor:
    """mkFlags k shape (corpus/c2_filter_sgmsum.ixl): int64 flag array of length k."""
    shape = _contig(shape.to(torch.int64))
    m = shape.numel()
    k = max(int(k), 0)
    out = torch.empty(k, dtype=torch.int64, device=shape.device)
    ws, wsb = _ws(L.OP_MKFLAGS, k, m, shape.device)
    L.check(_lib().ixg_mkflags(k, _ptr(shape), m, _ptr(out), variant, status.ptr, ws, wsb, _stream()), "mkflags")
    return out


def flag_bitmap(shape: torch.Tensor, nbits: int, d_nbits=None, bits=None, d_lo=None) -> torch.Tensor:
    """mkFlags over nbits output positions as a bitmap (int32 words); with
    d_nbits, over the device count (nbits is then the capacity); with d_lo
    (a device int64), over the window of positions [*d_lo, *d_lo + nbits)."""
    shape = _contig(shape.to(torch.int64))
    words = int(_lib().ixg_bitmap_words(nbits))
    if bits is None or bits.numel() < words:
        bits = torch.empty(words, dtype=torch.int32, device=shape.device)
    ws, wsb = _ws(L.OP_SCAN, shape.numel(), 0, shape.device)
    if d_lo is None:
        rc = _lib().ixg_flag_bitmap(_ptr(shape), shape.numel(), _ptr(bits), nbits, _ptr(d_nbits), ws, wsb, _stream())
    else:
        rc = _lib().ixg_flag_bitmap_window(_ptr(shape), shape.numel(), _ptr(bits), nbits, _ptr(d_nbits), _ptr(d_lo),
                                           ws, wsb, _stream())
    L.check(rc, "flag_bitmap")
    return bits


def segsum(vs: torch.Tensor, n: int, bits: torch.Tensor, flag_base: int, zs: torch.Tensor, carry_v: int,
           carry_f: bool, d_total: torch.Tensor, status: Status, d_n=None, d_flag_base=None):
    """zs[0..n) = sgmSum over vs with flags bits[flag_base + j] (ixg_segsum);
    d_n / d_flag_base: the same read from the device (n is then a capacity)."""
    ws, wsb = _ws(L.OP_SEGSCAN, vs.numel(), 0, vs.device)
    L.check(
        _lib().ixg_segsum(_dt(vs), _ptr(vs), n, _ptr(d_n), _ptr(bits), flag_base, _ptr(d_flag_base), _dt(zs), _ptr(zs),
                          carry_v, int(carry_f), _ptr(d_total), status.ptr, ws, wsb, _stream()),
        "segsum",
    )
    return zs


def seg_carry(bits: torch.Tensor, flag_base: int, zs: torch.Tensor, n: int, carry_v: int, scratch: torch.Tensor,
              status: Status, d_n=None, d_flag_base=None, d_aggs=None, rank: int = 0):
    """zs[q] += carry for q before the first flag of [flag_base, flag_base + n);
    carry = carry_v, or folded on the device from d_aggs (every rank's
    segmented aggregate) for `rank`."""
    L.check(
        _lib().ixg_seg_carry(_ptr(bits), flag_base, _ptr(d_flag_base), _dt(zs), _ptr(zs), n, _ptr(d_n), carry_v,
                             _ptr(d_aggs), rank, _ptr(scratch), status.ptr, _stream()),
        "seg_carry",
    )
    return zs


def _arr(t: torch.Tensor) -> L.ixg_array:
    return L.ixg_array(t.data_ptr() if t.numel() else 0, t.numel(), _dt(t), 0)


def map_vm(compiled, n: int, status: Status, stmt: int = 0, out_dtype=torch.int64, device=None) -> torch.Tensor:
    """map f xs... with a lambda compiled by vm.compile_map (oracle.py:274-280)."""
    out = torch.empty(n, dtype=out_dtype, device=device or torch.device("cuda"))
    ins = [_contig(t) for t in compiled.inputs]
    prog = (L.ixg_vm_insn * max(len(compiled.insns), 1))(*[L.ixg_vm_insn(op, d, a, b, c, 0, imm)
                                                          for op, d, a, b, c, imm in compiled.insns])
    arr_in = (L.ixg_array * max(len(ins), 1))(*[_arr(t) for t in ins])
    arr_out = (L.ixg_array * 1)(_arr(out))
    preds = (L.ixg_pred * max(len(compiled.preds), 1))(*[_c_pred(p) for p in compiled.preds])
    L.check(
        _lib().ixg_map(prog, len(compiled.insns), arr_in, len(ins), arr_out, 1, preds, len(compiled.preds), n, stmt,
                       status.ptr, _stream()),
        "map",
    )
    return out


def csr_gather(x: torch.Tensor, values: torch.Tensor, indices: torch.Tensor, variant: int, status: Status, out=None):
    """map2 (\\v c -> v * x[c]) values indices (corpus/c4_csr_gather.ixl)."""
    x, values, indices = _contig(x), _contig(values), _contig(indices)
    out = torch.empty(values.numel(), dtype=values.dtype, device=values.device) if out is None else out
    L.check(
        _lib().ixg_csr_gather(_dt(values), _ptr(x), x.numel(), _ptr(values), _ptr(indices), values.numel(), _ptr(out),
                              variant, status.ptr, _stream()),
        "csr_gather",
    )
    return out


def kmeans_ker(rows: torch.Tensor, pointers, cluster, values, indices, variant: int, status: Status):
    """kmeans_ker for each row in `rows` (corpus kmeans_ker.ixl)."""
    rows, pointers, indices = _contig(rows), _contig(pointers), _contig(indices)
    cluster, values = _contig(cluster.to(torch.float64)), _contig(values.to(torch.float64))
    out = torch.empty(rows.numel(), dtype=torch.float64, device=rows.device)
    L.check(
        _lib().ixg_kmeans_ker(_ptr(rows), rows.numel(), _ptr(pointers), pointers.numel(), _ptr(cluster),
                              cluster.numel(), _ptr(values), _ptr(indices), indices.numel(), _ptr(out), variant,
                              status.ptr, _stream()),
        "kmeans_ker",
    )
    return out


def eq_gather(H: torch.Tensor, es: torch.Tensor, is_: torch.Tensor, variant: int, status: Status, stmt: int = 0):
    """cs[i] = H[es[i]] == is[i] (maxmatching.ixl:18)."""
    H, es, is_ = _contig(H), _contig(es), _contig(is_)
    cs = torch.empty(es.numel(), dtype=torch.uint8, device=es.device)
    L.check(
        _lib().ixg_eq_gather(_ptr(H), H.numel(), _ptr(es), _ptr(is_), es.numel(), _ptr(cs), variant, stmt, status.ptr,
                             _stream()),
        "eq_gather",
    )
    return cs


def gen_uniform(n: int, lo: int, hi: int, seed: int, dtype=torch.int32, offset: int = 0, device=None, out=None):
    """Device-side counter-based input, identical to gen.uniform()."""
    out = torch.empty(n, dtype=dtype, device=device or torch.device("cuda")) if out is None else out
    L.check(_lib().ixg_gen_uniform(_dt(out), _ptr(out), n, lo, hi, seed, offset, _stream()), "gen_uniform")
    return out


def launch_count() -> int:
    return int(_lib().ixg_launch_count())


# ------------------------------------------------------------------ preconditions
def minmax(xs: torch.Tensor) -> torch.Tensor:
    """[min, max] of an integer array as a device int64 pair (ixg_minmax)."""
    xs = _contig(xs.view(torch.uint8) if xs.dtype == torch.bool else xs)
    out = torch.empty(2, dtype=torch.int64, device=xs.device)
    L.check(_lib().ixg_minmax(_dt(xs), _ptr(xs), xs.numel(), _ptr(out), _stream()), "minmax")
    return out


def mono_violations(xs: torch.Tensor, op: int) -> torch.Tensor:
    """adjacent pairs of xs violating op (0 <=, 1 <, 2 >=, 3 >) (ixg_mono_check)."""
    xs = _contig(xs)
    out = torch.empty(1, dtype=torch.int64, device=xs.device)
    L.check(_lib().ixg_mono_check(_dt(xs), _ptr(xs), xs.numel(), op, _ptr(out), _stream()), "mono_check")
    return out


def inj_check(xs: torch.Tensor, lo: int, hi: int, img_lo: int, img_hi: int) -> Optional[torch.Tensor]:
    """[in-range count, repeats, in-range values outside the image] over the
    values of xs in [lo, hi] (ixg_inj_check); None if the range is too wide
    for a claim bitmap."""
    xs = _contig(xs.to(torch.int64))
    nb = int(_lib().ixg_inj_bitmap_bytes(lo, hi))
    if nb < 0:
        return None
    bitmap = torch.empty(max(nb, 16), dtype=torch.uint8, device=xs.device)
    out = torch.empty(3, dtype=torch.int64, device=xs.device)
    L.check(_lib().ixg_inj_check(_ptr(xs), xs.numel(), lo, hi, img_lo, img_hi, _ptr(bitmap), bitmap.numel(), _ptr(out),
                                 _stream()), "inj_check")
    return out

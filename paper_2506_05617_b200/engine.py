"""Device orchestration of the LFA hot path over the C-ABI.

PyTorch is used only as plumbing here: device memory (caching allocator),
the current CUDA stream, events and torch.distributed.  Every byte of
compute is one of the library's sm_100a kernels, reached through _lib:

    K1  cs_symbol_field        half-grid symbol assembly
    K2/3 cs_batched_svd(_grouped)  one-sided Jacobi + per-block epilogue
    cs_complete_zero_columns / cs_first_failure / cs_spectrum_values

All tensors stay on the device; host copies happen only where the drop-in
API returns numpy arrays.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import AllocationFailure, ConvergenceFailure

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

DEFAULT_MAX_SWEEPS = 100   # blocksvd.py:25
DEFAULT_SVD_TOL = 1e-13    # blocksvd.py:26


def require_cuda(device=None):
    """Resolve the target device; fail loudly without CUDA (no CPU fallback)."""
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("convspectra_b200 needs a CUDA device (B200); no CPU fallback exists")
    _lib.load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"convspectra_b200 computes on CUDA devices only, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def dtype_code(dtype: str) -> int:
    if dtype == "f32":
        return _lib.CS_F32
    if dtype == "f64":
        return _lib.CS_F64
    raise ValueError(f"unknown dtype {dtype!r} (expected 'f32' or 'f64')")


def real_dtype(dtype: str):
    return torch.float32 if dtype == "f32" else torch.float64


def complex_dtype(dtype: str):
    return torch.complex64 if dtype == "f32" else torch.complex128


def dtype_of_tensor(t) -> str:
    if t.dtype in (torch.complex64, torch.float32):
        return "f32"
    return "f64"


TOL32_FLOOR = 2.5e-6


def check_tol(tol: float, dtype: str, rows: int) -> None:
    """Warn when a caller-supplied tolerance cannot be honoured in fp32.

    The reference default (1e-13, passed implicitly as DEFAULT_SVD_TOL) is
    floored silently in fp32 mode; an explicit value below the fp32
    resolution floor is floored too, but with a warning."""
    if dtype != "f32" or tol is DEFAULT_SVD_TOL:
        return
    floor = TOL32_FLOOR * math.sqrt(max(rows, 1) / 64.0)
    if float(tol) < floor:
        import warnings

        warnings.warn(f"tol={tol:g} is below the fp32 resolution floor {floor:.3g} for {rows}-row "
                      f"blocks; the fp32 solve uses {floor:.3g} (pass dtype='f64' for tighter "
                      "tolerances)", RuntimeWarning, stacklevel=3)


def effective_tol(tol: float, dtype: str, rows: int) -> float:
    """Convergence threshold actually used by the kernel.

    fp64 uses the caller's tol (reference default 1e-13, blocksvd.py:26).
    fp32 cannot resolve |gamma|/sqrt(alpha*beta) below its rounding floor
    (~eps32*sqrt(rows)); the threshold is floored at 2.5e-6*sqrt(rows/64) so
    the sweep loop terminates.  Measured on cfg5 (B200, tools/warmtest.py):
    floor 2e-6 -> 5.56 mean warm sweeps, 5e-6 -> 5.33, 1e-5 -> 5.24, with
    per-frequency sigma error 6-7e-7 of sigma_max in all three (bar 1e-5); the
    middle value keeps the threshold at half the bar."""
    if dtype == "f64":
        return float(tol)
    return max(float(tol), TOL32_FLOOR * math.sqrt(max(rows, 1) / 64.0))


def stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    """Raw device address for the C-ABI.  A lazily conjugated / negated torch
    view shares the unconjugated storage, so handing its address to a kernel
    would silently drop the conjugation: refuse it."""
    if t is None:
        return 0
    if t.is_conj() or t.is_neg():
        raise ValueError("lazily conjugated tensor passed to the C-ABI (call resolve_conj() first)")
    return t.data_ptr()


class _Workspace:
    """Grow-only device scratch per (device, stream) (the C-ABI owns no
    memory).  Keyed by the current stream so solves on different streams never
    share scratch; growth frees the old buffer through the caching allocator,
    which is stream-ordered on that same stream."""

    def __init__(self):
        self._buf = {}

    def get(self, device, nbytes: int):
        if nbytes <= 0:
            return None
        key = (device.type, device.index, torch.cuda.current_stream(device).cuda_stream)
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            self._buf[key] = None
            buf = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
            self._buf[key] = buf
        return buf


WORKSPACE = _Workspace()


def half_grid_count(n: int, m: int) -> int:
    """Conjugate-orbit representatives, same as cs_half_grid_count."""
    h0 = m // 2 + 1
    nmid = (n - 1) // 2
    return h0 + nmid * m + (h0 if (n % 2 == 0 and n > 1) else 0)


def half_grid_indices(n: int, m: int) -> np.ndarray:
    """Full-grid index f of each representative, in representative order."""
    h0 = m // 2 + 1
    rows = [np.arange(h0)]
    for i in range(1, (n - 1) // 2 + 1):
        rows.append(i * m + np.arange(m))
    if n % 2 == 0 and n > 1:
        rows.append((n // 2) * m + np.arange(h0))
    return np.concatenate(rows).astype(np.int64)


def partner_map(n: int, m: int):
    """For each full-grid f: (representative index u, conj flag)."""
    f = np.arange(n * m)
    i, j = f // m, f % m
    fs = ((n - i) % n) * m + (m - j) % m
    rep = f <= fs
    frep = np.where(rep, f, fs)
    reps = half_grid_indices(n, m)
    lut = np.full(n * m, -1, dtype=np.int64)
    lut[reps] = np.arange(len(reps))
    return lut[frep], ~rep


def self_conjugate_count(n: int, m: int) -> int:
    return (1 + (n % 2 == 0)) * (1 + (m % 2 == 0))


# ---------------------------------------------------------------------------
# K1
# ---------------------------------------------------------------------------
def weights_to_device(kernel, dtype: str, device):
    w = kernel.device_weights(dtype)
    return torch.from_numpy(w).to(device, non_blocking=False)


def symbol_field(w_dev, dims_n: int, dims_m: int, dtype: str, half: bool = True,
                 f_first: int = 0, f_count: int | None = None, out=None, layout: int = 0):
    """Symbol blocks for a contiguous range of (representative or full-grid) frequencies."""
    co, ci, kh, kw = w_dev.shape
    total = half_grid_count(dims_n, dims_m) if half else dims_n * dims_m
    if f_count is None:
        f_count = total - f_first
    if out is None:
        shape = (f_count, co, ci) if layout == 0 else (co, ci, f_count)
        out = torch.empty(shape, dtype=complex_dtype(dtype), device=w_dev.device)
    st = _lib.load().cs_symbol_field(ptr(w_dev), dtype_code(dtype), co, ci, kh, kw, dims_n,
                                     dims_m, f_first, f_count, int(half), ptr(out), layout,
                                     stream_ptr(w_dev.device))
    _lib.check(st, "cs_symbol_field")
    return out


def fft_symbol_field(w_dev, dims_n: int, dims_m: int, dtype: str, half: bool = True,
                     timer=None, out=None):
    """Symbol blocks by the FFT route (cs_fft_transform + cs_fft_gather):
    embed, batched 2D DFT per channel pair, gather.  ``timer`` gets a mark
    "tf" between the transform and the gather (s_transform | s_copy)."""
    co, ci, kh, kw = w_dev.shape
    total = half_grid_count(dims_n, dims_m) if half else dims_n * dims_m
    lib = _lib.load()
    nbytes = lib.cs_fft_field_workspace(dtype_code(dtype), co, ci, dims_n, dims_m)
    emb = torch.empty(int(nbytes), dtype=torch.uint8, device=w_dev.device)
    st = stream_ptr(w_dev.device)
    _lib.check(lib.cs_fft_transform(ptr(w_dev), dtype_code(dtype), co, ci, kh, kw, dims_n, dims_m,
                                    ptr(emb), nbytes, st), "cs_fft_transform")
    if timer:
        timer.mark("tf")
    if out is None:
        out = torch.empty((total, co, ci), dtype=complex_dtype(dtype), device=w_dev.device)
    _lib.check(lib.cs_fft_gather(ptr(emb), dtype_code(dtype), co, ci, dims_n, dims_m, int(half),
                                 ptr(out), st), "cs_fft_gather")
    del emb  # stream-ordered reuse by the caching allocator
    return out


def symbol_at_freqs(w_dev, freqs: np.ndarray, dtype: str):
    co, ci, kh, kw = w_dev.shape
    fr = torch.from_numpy(np.ascontiguousarray(freqs, dtype=np.float64)).to(w_dev.device)
    out = torch.empty((len(freqs), co, ci), dtype=complex_dtype(dtype), device=w_dev.device)
    st = _lib.load().cs_symbol_at(ptr(w_dev), dtype_code(dtype), co, ci, kh, kw, ptr(fr),
                                  len(freqs), ptr(out), stream_ptr(w_dev.device))
    _lib.check(st, "cs_symbol_at")
    return out


def expand_half(half, n: int, m: int, dtype: str, out=None):
    F_u, a, b = half.shape
    if out is None:
        out = torch.empty((n * m, a, b), dtype=half.dtype, device=half.device)
    st = _lib.load().cs_expand_half_grid(ptr(half), dtype_code(dtype), a, b, n, m, ptr(out),
                                         stream_ptr(half.device))
    _lib.check(st, "cs_expand_half_grid")
    return out


def is_conj_symmetric(full, n: int, m: int, dtype: str) -> bool:
    F, a, b = full.shape
    flag = torch.empty(1, dtype=torch.int32, device=full.device)
    st = _lib.load().cs_check_conj_symmetry(ptr(full), dtype_code(dtype), a, b, n, m, ptr(flag),
                                            stream_ptr(full.device))
    _lib.check(st, "cs_check_conj_symmetry")
    return bool(flag.item())


# ---------------------------------------------------------------------------
# K2/K3
# ---------------------------------------------------------------------------
@dataclass
class SvdBatch:
    sigma: "torch.Tensor"          # (count, r) descending, real
    info: "torch.Tensor"           # (count,) int32 sweeps or -1
    U: "torch.Tensor | None" = None  # (count, c_out, r)
    V: "torch.Tensor | None" = None  # (count, c_in, r)
    zero: "torch.Tensor | None" = None


def alloc_svd_outputs(count, co, ci, dtype, want_vectors, device):
    r = min(co, ci)
    sig = torch.empty((count, r), dtype=real_dtype(dtype), device=device)
    info = torch.empty((count,), dtype=torch.int32, device=device)
    U = V = zero = None
    if want_vectors:
        U = torch.empty((count, co, r), dtype=complex_dtype(dtype), device=device)
        V = torch.empty((count, ci, r), dtype=complex_dtype(dtype), device=device)
        zero = torch.empty((count,), dtype=torch.int32, device=device)
    return SvdBatch(sig, info, U, V, zero)


def batched_svd(blocks, dtype: str, want_vectors: bool, tol=DEFAULT_SVD_TOL,
                max_sweeps=DEFAULT_MAX_SWEEPS, out: SvdBatch | None = None,
                complete=True) -> SvdBatch:
    """SVD of every (c_out, c_in) block of a contiguous device tensor."""
    count, co, ci = blocks.shape
    dev = blocks.device
    lib = _lib.load()
    if out is None:
        out = alloc_svd_outputs(count, co, ci, dtype, want_vectors, dev)
    code = dtype_code(dtype)
    ws_bytes = lib.cs_batched_svd_workspace(code, count, co, ci, int(want_vectors))
    ws = WORKSPACE.get(dev, ws_bytes)
    etol = effective_tol(tol, dtype, max(co, ci))
    st = lib.cs_batched_svd(ptr(blocks), code, count, co, ci, int(want_vectors), etol,
                            int(max_sweeps), ptr(out.sigma), ptr(out.U), ptr(out.V),
                            ptr(out.info), ptr(out.zero), ptr(ws), ws_bytes, stream_ptr(dev))
    _lib.check(st, "cs_batched_svd")
    if want_vectors and complete:
        complete_zero_columns(out, co, ci, dtype)
    return out


def batched_svd_grouped(groups, dtype: str, want_vectors: bool, tol=DEFAULT_SVD_TOL,
                        max_sweeps=DEFAULT_MAX_SWEEPS):
    """One call over heterogeneous layers: groups = [blocks tensor, ...]."""
    lib = _lib.load()
    outs = []
    table = (_lib.SvdGroup * len(groups))()
    dev = groups[0].device
    rows = 1
    # the library forks groups onto streams in table order: the costliest
    # (count * mr * nc^2) first, so the long large-block solves start while
    # the SMs are free and the small ones fill in around them
    def cost(blk):
        count, co, ci = blk.shape
        return count * max(co, ci) * min(co, ci) ** 2
    order = sorted(range(len(groups)), key=lambda g: -cost(groups[g]))
    for blk in groups:
        count, co, ci = blk.shape
        outs.append(alloc_svd_outputs(count, co, ci, dtype, want_vectors, dev))
        rows = max(rows, co, ci)
    for slot, g in enumerate(order):
        blk, o = groups[g], outs[g]
        count, co, ci = blk.shape
        table[slot] = _lib.SvdGroup(ptr(blk), count, co, ci, ptr(o.sigma), ptr(o.U), ptr(o.V),
                                    ptr(o.info), ptr(o.zero), effective_tol(tol, dtype, max(co, ci)))
    code = dtype_code(dtype)
    ws_bytes = lib.cs_batched_svd_grouped_workspace(table, len(groups), code, int(want_vectors))
    ws = WORKSPACE.get(dev, ws_bytes)
    etol = effective_tol(tol, dtype, rows)  # per-group tols override it
    st = lib.cs_batched_svd_grouped(table, len(groups), code, int(want_vectors), etol,
                                    int(max_sweeps), ptr(ws), ws_bytes, stream_ptr(dev))
    _lib.check(st, "cs_batched_svd_grouped")
    if want_vectors:
        for blk, o in zip(groups, outs):
            complete_zero_columns(o, blk.shape[1], blk.shape[2], dtype)
    return outs


def plan_kind(count: int, co: int, ci: int, dtype: str, want_vectors: bool) -> int:
    return int(_lib.load().cs_batched_svd_plan_kind(dtype_code(dtype), count, co, ci,
                                                    int(want_vectors)))


def batched_svd_indexed(blocks, dtype: str, want_vectors: bool, index, out: SvdBatch,
                        tol=DEFAULT_SVD_TOL, max_sweeps=DEFAULT_MAX_SWEEPS, init_X=None,
                        init_V=None, init_V_index=None, plan_count: int = 0):
    """Solve blocks[index[i]] (outputs at index[i]; index None: all blocks);
    optional warm start from init_X[i] / init_V[init_V_index[i]]
    (cs_batched_svd_indexed).  plan_count > 0 fixes the kernel configuration
    to that of a plan_count-matrix batch (shard-independent results)."""
    _, co, ci = blocks.shape
    count = index.shape[0] if index is not None else blocks.shape[0]
    dev = blocks.device
    lib = _lib.load()
    code = dtype_code(dtype)
    ws_bytes = lib.cs_batched_svd_workspace(code, max(count, int(plan_count)), co, ci, int(want_vectors))
    ws = WORKSPACE.get(dev, ws_bytes)
    etol = effective_tol(tol, dtype, max(co, ci))
    st = lib.cs_batched_svd_indexed(ptr(blocks), code, count, co, ci, int(want_vectors), etol,
                                    int(max_sweeps), ptr(index), ptr(init_X), ptr(init_V),
                                    ptr(init_V_index), int(plan_count), ptr(out.sigma), ptr(out.U),
                                    ptr(out.V), ptr(out.info), ptr(out.zero), ptr(ws), ws_bytes,
                                    stream_ptr(dev))
    _lib.check(st, "cs_batched_svd_indexed")
    return out


def warm_start_gemm(blocks, dtype: str, warm_ids, seed_ids, Vw, out_X):
    _, co, ci = blocks.shape
    st = _lib.load().cs_warm_start_gemm(ptr(blocks), dtype_code(dtype), co, ci,
                                        warm_ids.shape[0], ptr(warm_ids), ptr(seed_ids),
                                        ptr(Vw), ptr(out_X), stream_ptr(blocks.device))
    _lib.check(st, "cs_warm_start_gemm")
    return out_X


_WARM_PLANS = {}
_WARM_DEPTH_ENV = os.environ.get("CS_WARM_DEPTH")


def warm_depth(count: int) -> int:
    """Seed lattice half-period: deep chains (few cold seeds) pay when there
    are many blocks per stage, short ones (few staged launches) otherwise.
    Measured: cfg5 (32770 blocks) warm SVD depth 3 -> 4.83 s, 5 -> 4.74,
    8 -> 4.72, 12 -> 4.74, 24 -> 4.77; cfg2 (2050) step depth 3 -> 6.94 ms,
    8 -> 9.05 ms (cold 7.83); cfg3 (1570) depth 2/3 -> 59.1 ms, 5 -> 62.6,
    8 -> 68.8 (cold 78.0)."""
    if _WARM_DEPTH_ENV is not None:
        return int(_WARM_DEPTH_ENV)
    return 8 if count >= 16384 else 3


WARM_DEPTH = int(_WARM_DEPTH_ENV) if _WARM_DEPTH_ENV is not None else 3  # warm_plan() default (no block shape)


def _bfs_forest(n: int, m: int, u0: int, count: int, depth: int):
    """Host BFS forest over representatives [u0, u0+count): (level, parent)
    with parent as a local index (-1 for seeds)."""
    reps = half_grid_indices(n, m)[u0:u0 + count]
    ii, jj = reps // m, reps % m
    local = {(int(a), int(b)): q for q, (a, b) in enumerate(zip(ii, jj))}
    span = 2 * depth + 1
    level = np.full(count, -1, dtype=np.int64)
    parent = np.full(count, -1, dtype=np.int64)
    frontier = [q for q in range(count) if ii[q] % span == depth % span and jj[q] % span == depth]
    if not frontier:
        frontier = [0]
    for q in frontier:
        level[q] = 0
    while True:
        while frontier:
            nxt = []
            for q in frontier:
                a, b = int(ii[q]), int(jj[q])
                for nb in ((a, b - 1), (a, b + 1), (a - 1, b), (a + 1, b)):
                    r = local.get(nb)
                    if r is not None and level[r] < 0:
                        level[r] = level[q] + 1
                        parent[r] = q
                        nxt.append(r)
            frontier = nxt
        left = np.nonzero(level < 0)[0]
        if len(left) == 0:
            break
        level[left[0]] = 0
        frontier = [int(left[0])]
    return level, parent


_FORESTS = {}


def warm_forest(n: int, m: int, depth: int | None = None):
    """The warm-start forest over ALL representatives of an n x m grid:
    (level, parent, root) per representative (global indices).  A frequency
    shard made of whole trees solves every block exactly as the single-GPU
    plan does (same seed, same parent chain)."""
    total = half_grid_count(n, m)
    depth = warm_depth(total) if depth is None else depth
    key = (n, m, depth)
    if key not in _FORESTS:
        level, parent = _bfs_forest(n, m, 0, total, depth)
        root = np.arange(total, dtype=np.int64)
        for q in np.argsort(level, kind="stable"):  # parents sit one level earlier
            if parent[q] >= 0:
                root[q] = root[parent[q]]
        _FORESTS[key] = (level, parent, root)
    return _FORESTS[key]


def warm_plan(n: int, m: int, u0: int, count: int, device, depth: int | None = None):
    """Stages of a warm-started solve over representatives [u0, u0+count).

    Representatives are nodes of the frequency lattice (i, j); two are
    neighbours when they differ by one grid step in i or j (their symbols
    differ by O(2 pi/n) relatively).  Cold seeds sit on a (2*depth+1)-periodic
    lattice; a breadth-first search from the seeds assigns every other
    representative to the stage equal to its lattice distance, warm-started
    from its BFS parent (solved one stage earlier).  Representatives not
    reachable within the range become seeds.  Returns [(ids, pred_or_None)]
    per stage as device int64 tensors of local indices."""
    depth = WARM_DEPTH if depth is None else depth
    key = (n, m, u0, count, str(device), depth)
    if key in _WARM_PLANS:
        return _WARM_PLANS[key]
    level, parent = _bfs_forest(n, m, u0, count, depth)
    t = lambda x: torch.tensor(np.asarray(x, dtype=np.int64), device=device)
    plan = []
    for d in range(int(level.max()) + 1):
        ids = np.nonzero(level == d)[0]
        if len(ids):
            plan.append((t(ids), t(parent[ids]) if d else None))
    _WARM_PLANS[key] = plan
    return plan


def subset_plan(n: int, m: int, ids, device, depth: int | None = None):
    """Stages of the global warm forest restricted to the representatives
    `ids` (sorted; whole trees): [(local ids, local parents or None, global
    stage size)].  The global stage size is the plan_count that keeps each
    stage's kernel configuration that of the single-GPU solve."""
    level, parent, _ = warm_forest(n, m, depth)
    ids = np.asarray(ids, dtype=np.int64)
    pos = np.full(len(level), -1, dtype=np.int64)
    pos[ids] = np.arange(len(ids))
    lv = level[ids]
    t = lambda x: torch.tensor(np.asarray(x, dtype=np.int64), device=device)
    plan = []
    for d in range(int(level.max()) + 1):
        sel = np.nonzero(lv == d)[0]
        if len(sel) == 0:
            continue
        gsize = int(np.count_nonzero(level == d))
        if d == 0:
            plan.append((t(sel), None, gsize))
        else:
            par = pos[parent[ids[sel]]]
            if (par < 0).any():
                raise ValueError("a shard must consist of whole warm-start trees")
            plan.append((t(sel), t(par), gsize))
    return plan


def batched_svd_warm(blocks, dtype: str, n: int, m: int, u0: int, tol=DEFAULT_SVD_TOL,
                     max_sweeps=DEFAULT_MAX_SWEEPS, depth: int | None = None, ids=None):
    """All blocks of a representative range (or of the representative set
    `ids` -- whole warm-start trees -- with `blocks` in that order); every
    non-seed block is warm-started from its solved neighbour's right factor
    (cs_warm_start_gemm + cs_batched_svd_indexed), stage by stage.  Each
    stage is planned for its size in the whole grid's forest, so a shard's
    blocks come out bit for bit as in the single-GPU solve."""
    count, co, ci = blocks.shape
    dev = blocks.device
    if ids is not None or u0 == 0 and count == half_grid_count(n, m):
        sel_ids = np.arange(count) if ids is None else ids
        stages = subset_plan(n, m, sel_ids, dev, depth)
    else:
        if depth is None:
            depth = warm_depth(count)
        stages = [(i, p, 0) for i, p in warm_plan(n, m, u0, count, dev, depth)]
    out = alloc_svd_outputs(count, co, ci, dtype, True, dev)
    wide = co < ci
    mr, nc = (ci, co) if wide else (co, ci)
    Vw = out.U if wide else out.V
    for sel, pred, gsize in stages:
        if pred is None:
            batched_svd_indexed(blocks, dtype, True, sel, out, tol, max_sweeps, plan_count=gsize)
        else:
            Xw = torch.empty((sel.shape[0], mr, nc), dtype=blocks.dtype, device=dev)
            warm_start_gemm(blocks, dtype, sel, pred, Vw, Xw)
            batched_svd_indexed(blocks, dtype, True, sel, out, tol, max_sweeps, init_X=Xw,
                                init_V=Vw, init_V_index=pred, plan_count=gsize)
            del Xw
    complete_zero_columns(out, co, ci, dtype)
    return out


def use_warm_start(count: int, co: int, ci: int, dtype: str, want_vectors: bool,
                   requested=None) -> bool:
    """Warm start pays off when vectors are computed anyway (seeds need V)
    and the blocks are not tiny: 16 x 16 blocks converge cold in ~7 cheap
    sweeps, and the staged warm launches cost more than they save (cfg1:
    3.3 ms per call warm vs ~1 ms cold).  CS_WARM_START=0/1 forces it."""
    env = os.environ.get("CS_WARM_START")
    if requested is None:
        requested = (env != "0") if env is not None else (want_vectors and min(co, ci) >= 32)
    if not requested or count < 3:
        return False
    return plan_kind(count, co, ci, dtype, True) == 2


def values_via_vectors(count: int, co: int, ci: int, dtype: str) -> bool:
    """Whether a values-only drop-in call runs the vectors solve (factors
    dropped): yes whenever the vectors solve is the panel / tensor-core
    kernel, so values_only=True and False agree bit for bit.  Shapes whose
    vectors solve needs the generic fallback kernel keep the faster
    values-only kernel (values then agree to fp rounding, not bitwise)."""
    return count > 0 and plan_kind(count, co, ci, dtype, True) == 2


def use_warm_values(count: int, co: int, ci: int, dtype: str) -> bool:
    """Values-only solve of tall blocks through the warm-started vectors path
    (U/V computed and dropped): with nc <= mr/2 the V rows cost at most half
    the X rows, and the warm start halves the sweeps (cfg3 256x128).
    CS_WARM_VALUES=0 disables."""
    if os.environ.get("CS_WARM_VALUES") == "0" or dtype != "f32" or count < 3:
        return False
    mr, nc = max(co, ci), min(co, ci)
    return nc >= 64 and mr >= 2 * nc and plan_kind(count, co, ci, dtype, True) == 2


def complete_zero_columns(out: SvdBatch, co: int, ci: int, dtype: str):
    """blocksvd.py:184-198 on the factor of the working (tall) matrix."""
    if out.zero is None or out.sigma.shape[0] == 0:
        return
    wide = co < ci
    Uw = out.V if wide else out.U
    mr = ci if wide else co
    r = min(co, ci)
    st = _lib.load().cs_complete_zero_columns(ptr(Uw), dtype_code(dtype), out.sigma.shape[0], mr,
                                              r, ptr(out.sigma), ptr(out.zero),
                                              stream_ptr(out.sigma.device))
    _lib.check(st, "cs_complete_zero_columns")


def first_failure(info) -> int:
    first = torch.empty(1, dtype=torch.int64, device=info.device)
    st = _lib.load().cs_first_failure(ptr(info), info.shape[0], ptr(first),
                                      stream_ptr(info.device))
    _lib.check(st, "cs_first_failure")
    return int(first.item())


def spectrum_values(sigma, dtype: str, n: int, m: int, half: bool):
    """Flat descending float64 values on the device (conj partners duplicated)."""
    count, r = sigma.shape
    nv = n * m * r if half else count * r
    lib = _lib.load()
    code = dtype_code(dtype)
    ws_bytes = lib.cs_spectrum_values_workspace(nv, code)
    ws = WORKSPACE.get(sigma.device, ws_bytes)
    values = torch.empty((nv,), dtype=torch.float64, device=sigma.device)
    st = lib.cs_spectrum_values(ptr(sigma), code, count, r, n, m, int(half), ptr(values), ptr(ws),
                                ws_bytes, stream_ptr(sigma.device))
    _lib.check(st, "cs_spectrum_values")
    return values


def raise_convergence(f: int, freqs=None, max_sweeps=DEFAULT_MAX_SWEEPS):
    """Reference message shape of blocksvd.py:213-224."""
    where = f"block {f}"
    if freqs is not None:
        k = freqs[f]
        where = f"frequency index {f} (k=({k[0]:.6g}, {k[1]:.6g}))"
    raise ConvergenceFailure(
        f"jacobi SVD did not converge within {max_sweeps} sweeps at {where}; "
        "check the input for NaN/Inf contamination")


def device_budget_bytes(device, mem_budget_gib=None) -> int:
    """Field budget for device-resident paths: the explicit parameter, then the
    reference's env knob, else the device's total memory."""
    if mem_budget_gib is not None:
        return int(float(mem_budget_gib) * 2**30)
    env = os.environ.get("CONV_SPECTRA_MEM_BUDGET_GIB")
    if env is not None:
        return int(float(env) * 2**30)
    return int(torch.cuda.get_device_properties(device).total_memory)


def check_budget(need: int, budget: int, what: str):
    if need > budget:
        raise AllocationFailure(f"{what} needs {need} bytes, budget is {budget} bytes")


class Timer:
    """CUDA-event phase timer on the current stream of `device`."""

    def __init__(self, device):
        self.device = device
        self.events = {}

    def mark(self, name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self.device))
        self.events[name] = ev

    def seconds(self, a, b) -> float:
        self.events[b].synchronize()
        return self.events[a].elapsed_time(self.events[b]) / 1e3


def materialize_vector(factor, col: int, fi: int, fj: int, n: int, m: int, dtype: str):
    rows, r = factor.shape
    out = torch.empty((n * m * rows,), dtype=complex_dtype(dtype), device=factor.device)
    st = _lib.load().cs_materialize_vector(ptr(factor.resolve_conj().contiguous()), dtype_code(dtype), rows, r,
                                           col, fi, fj, n, m, ptr(out),
                                           stream_ptr(factor.device))
    _lib.check(st, "cs_materialize_vector")
    return out


def apply_conv(w_dev, x, n: int, m: int, dtype: str):
    co, ci, kh, kw = w_dev.shape
    y = torch.empty((m, n, co), dtype=complex_dtype(dtype), device=w_dev.device)
    st = _lib.load().cs_apply_conv(ptr(w_dev), dtype_code(dtype), co, ci, kh, kw, n, m,
                                   ptr(x.contiguous()), ptr(y), stream_ptr(w_dev.device))
    _lib.check(st, "cs_apply_conv")
    return y


def fma_peak_flops(dtype: str = "f32", device_index: int = 0) -> float:
    """Measured FFMA/DFMA throughput (flop/s) for the roofline denominator."""
    return float(_lib.load().cs_measure_fma_peak(dtype_code(dtype), device_index))


_ = ctypes  # keep import for type users

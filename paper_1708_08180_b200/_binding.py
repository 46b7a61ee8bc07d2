"""Thin ctypes binding over libccl.so (include/ccl.h).  Argument marshalling
only: every step of the labeling runs in the library's CUDA kernels.  PyTorch
supplies device memory (caching allocator) and the current CUDA stream.

There is deliberately no fallback: if libccl.so is missing or cannot be
loaded, importing this module raises (build it with
``python paper_1708_08180_b200/_build.py`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import contextlib
import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libccl.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1708_08180_b200/_build.py` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

_i64, _int, _sz, _vp = ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/ccl.h
SIGNATURES = {
    "ccl_status_string": (ctypes.c_char_p, [_int]),
    "ccl_last_cuda_error": (_int, []),
    "ccl_workspace_bytes": (_sz, [_i64, _i64, _i64, _int]),
    "ccl_label": (_int, [_vp, _i64, _i64, _int, _vp]),
    "ccl_label_batched": (_int, [_vp, _i64, _i64, _i64, _int, _vp]),
    "ccl_label_batched_async": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp, _sz, _vp]),
    "ccl_label_batched_cfg_async": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp, _sz, _int, _vp]),
    "ccl_stage_local_merge": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _sz, _int, _vp]),
    "ccl_stage_boundary": (_int, [_i64, _i64, _i64, _int, _vp, _sz, _int, _vp]),
    "ccl_stage_link": (_int, [_i64, _i64, _i64, _int, _vp, _vp, _sz, _int, _vp]),
    "ccl_default_tile_rows": (_int, [_i64, _i64, _i64]),
    "ccl_label_threshold_async": (_int, [_vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _int, _vp]),
    "ccl_boundary_work_items": (_i64, [_i64, _i64, _i64, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "ccl_host_scratch_bytes": (_sz, [_i64, _i64, _i64, _int]),
    "ccl_label_host_async": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp, _sz, _vp]),
    "ccl_strip_workspace_bytes": (_sz, [_i64, _i64, _int, _int]),
    "ccl_strip_local": (_int, [_vp, _i64, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _sz, _vp]),
    "ccl_strip_finalize": (_int, [_vp, _int, _int, _i64, _i64, _i64, _i64, _int, _vp, _vp, _sz, _vp]),
    "ccl_method_workspace_bytes": (_sz, [_i64, _i64, _i64, _int, _int]),
    "ccl_stats_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "ccl_label_equal_async": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp, _sz, _vp]),
    "ccl_workspace_bytes_3d": (_sz, [_i64, _i64, _i64, _i64, _int]),
    "ccl_label_3d_async": (_int, [_vp, _i64, _i64, _i64, _i64, _int, _vp, _vp, _sz, _vp]),
    "ccl_component_stats_async": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "ccl_component_stats_relabel_async": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ccl_label_method_async": (_int, [_vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp]),
}

# the paper's comparison methods (include/ccl.h CCL_METHOD_*)
METHODS = {"optimized": 0, "uf": 1, "line_uf": 2, "le": 3}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

STATUS = {0: "CCL_OK", 1: "CCL_ERR_NULL", 2: "CCL_ERR_DIMS", 3: "CCL_ERR_TOO_LARGE",
          4: "CCL_ERR_CONNECTIVITY", 5: "CCL_ERR_ALIAS", 6: "CCL_ERR_WORKSPACE",
          7: "CCL_ERR_CUDA", 8: "CCL_ERR_CONFIG"}


class CCLError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        msg = _lib.ccl_status_string(status).decode()
        if status == 7:
            msg += f" (cudaError {_lib.ccl_last_cuda_error()})"
        super().__init__(f"{where}: {self.name}: {msg}")


def _check(status: int, where: str) -> None:
    if status != 0:
        raise CCLError(status, where)


def raw():
    """The underlying ctypes CDLL (tests call the C ABI through it)."""
    return _lib


def status_string(status: int) -> str:
    return _lib.ccl_status_string(status).decode()


def workspace_bytes(B: int, H: int, W: int, connectivity: int = 8) -> int:
    return int(_lib.ccl_workspace_bytes(B, H, W, connectivity))


def strip_workspace_bytes(rows: int, W: int, k: int, connectivity: int = 8) -> int:
    return int(_lib.ccl_strip_workspace_bytes(rows, W, k, connectivity))


def default_tile_rows(B: int, H: int, W: int) -> int:
    """The tile height tile_rows=0 selects for this geometry on the current device."""
    ty = _lib.ccl_default_tile_rows(B, H, W)
    if ty < 0:
        raise ValueError("invalid geometry")
    return int(ty)


def boundary_work_items(B: int, H: int, W: int, tile_rows: int = 0):
    h, v = _i64(0), _i64(0)
    total = _lib.ccl_boundary_work_items(B, H, W, tile_rows, ctypes.byref(h), ctypes.byref(v))
    if total < 0:
        raise ValueError("invalid geometry")
    return int(h.value), int(v.value)


def _torch():
    import torch
    return torch


def _shape3(t):
    if t.dim() == 2:
        return 1, int(t.shape[0]), int(t.shape[1])
    if t.dim() == 3:
        return int(t.shape[0]), int(t.shape[1]), int(t.shape[2])
    raise ValueError(f"expected [H,W] or [B,H,W], got shape {tuple(t.shape)}")


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@contextlib.contextmanager
def _on(device, stream=None):
    """Run a wrapper body on ``device``: it becomes the current device (the
    library launches on the current device), ``stream`` defaults to that
    device's current stream, and every temporary the body allocates belongs to
    that stream in the caching allocator (so a block is not handed to another
    stream while the library's kernels still use it)."""
    torch = _torch()
    device = torch.device(device)
    with torch.cuda.device(device):
        s = stream if stream is not None else torch.cuda.current_stream(device)
        if s.device != device:
            raise ValueError(f"stream is on {s.device}, the tensors on {device}")
        with torch.cuda.stream(s):
            yield s


def _same_device(device, *tensors):
    for t in tensors:
        if t is not None and t.device != device:
            raise ValueError(f"all tensors must be on {device}, got one on {t.device}")


def _check_out(out, shape, device):
    """A caller-supplied output: contiguous int32 of the input's shape, same device."""
    torch = _torch()
    if out.dtype != torch.int32 or tuple(out.shape) != tuple(shape) or not out.is_contiguous():
        raise ValueError("out must be a contiguous int32 tensor of the input's shape")
    _same_device(device, out)


def _check_image(image):
    torch = _torch()
    if not isinstance(image, torch.Tensor) or not image.is_cuda:
        raise TypeError("image must be a CUDA tensor (there is no CPU path)")
    if image.dtype != torch.uint8:
        raise TypeError(f"image must be uint8, got {image.dtype}")
    if not image.is_contiguous():
        raise ValueError("image must be contiguous (row-major, no pitch)")


class Workspace:
    """Reusable device workspace (a torch uint8 buffer) for repeated calls."""

    def __init__(self, B: int, H: int, W: int, connectivity: int = 8, device=None):
        torch = _torch()
        n = workspace_bytes(B, H, W, connectivity)
        if n == 0:
            raise ValueError("invalid geometry")
        self.nbytes = n
        self.buf = torch.empty(n, dtype=torch.uint8, device=device or "cuda")

    def ptr(self):
        return ctypes.c_void_p(self.buf.data_ptr())


def label(image, connectivity: int = 8, *, out=None, workspace: Workspace | None = None,
          tile_rows: int = 0, stream=None, threshold: int = 1):
    """Label a uint8 CUDA image [H,W] or batch [B,H,W]; returns int32 labels of
    the same shape (0 = background, 1 + min raster index per component, per
    image).  Foreground: value >= ``threshold`` (default 1: nonzero; another
    value runs ccl_label_threshold_async, the binarisation fused into K1).
    Enqueued on ``stream`` (default: torch's current stream)."""
    torch = _torch()
    _check_image(image)
    B, H, W = _shape3(image)
    with _on(image.device, stream) as s:
        if out is None:
            out = torch.empty(image.shape, dtype=torch.int32, device=image.device)
        else:
            _check_out(out, image.shape, image.device)
        if B == 0:
            return out
        if workspace is None:
            workspace = Workspace(B, H, W, connectivity, device=image.device)
        _same_device(image.device, workspace.buf)
        if threshold == 1:
            _check(_lib.ccl_label_batched_cfg_async(
                ctypes.c_void_p(image.data_ptr()), B, H, W, int(connectivity), ctypes.c_void_p(out.data_ptr()),
                workspace.ptr(), workspace.nbytes, int(tile_rows), _stream_ptr(s)), "ccl_label_batched_cfg_async")
        else:
            _check(_lib.ccl_label_threshold_async(
                ctypes.c_void_p(image.data_ptr()), B, H, W, int(connectivity), int(threshold),
                ctypes.c_void_p(out.data_ptr()), workspace.ptr(), workspace.nbytes, int(tile_rows),
                _stream_ptr(s)), "ccl_label_threshold_async")
    return out


class MethodWorkspace:
    """Device workspace for label_method (one of METHODS)."""

    def __init__(self, B: int, H: int, W: int, connectivity: int, method: str, device=None):
        torch = _torch()
        n = int(_lib.ccl_method_workspace_bytes(B, H, W, connectivity, METHODS[method]))
        if n == 0:
            raise ValueError("invalid geometry or method")
        self.nbytes = n
        self.buf = torch.empty(n, dtype=torch.uint8, device=device or "cuda")

    def ptr(self):
        return ctypes.c_void_p(self.buf.data_ptr())


def label_method(image, connectivity: int = 8, method: str = "uf", *, out=None,
                 workspace: MethodWorkspace | None = None, stream=None):
    """Label with one of the paper's comparison methods (conventional UF,
    line-based UF, label equivalence; or "optimized" = this library's path)
    through ccl_label_method_async.  Same canonical output as label()."""
    torch = _torch()
    _check_image(image)
    B, H, W = _shape3(image)
    if method not in METHODS:
        raise ValueError(f"method must be one of {sorted(METHODS)}")
    with _on(image.device, stream) as s:
        if out is None:
            out = torch.empty(image.shape, dtype=torch.int32, device=image.device)
        else:
            _check_out(out, image.shape, image.device)
        if B == 0:
            return out
        if workspace is None:
            workspace = MethodWorkspace(B, H, W, connectivity, method, device=image.device)
        _same_device(image.device, workspace.buf)
        _check(_lib.ccl_label_method_async(
            ctypes.c_void_p(image.data_ptr()), B, H, W, int(connectivity), METHODS[method],
            ctypes.c_void_p(out.data_ptr()), workspace.ptr(), workspace.nbytes, _stream_ptr(s)),
            "ccl_label_method_async")
    return out


def label_equal(image, connectivity: int = 8, *, out=None, stream=None):
    """Equal-value mode (NEXT-2, ccl_label_equal_async): every pixel labeled
    with the 0-based minimum raster index of its component of equal-valued
    pixels (background included; grey-level input allowed)."""
    torch = _torch()
    _check_image(image)
    B, H, W = _shape3(image)
    with _on(image.device, stream) as s:
        if out is None:
            out = torch.empty(image.shape, dtype=torch.int32, device=image.device)
        else:
            _check_out(out, image.shape, image.device)
        if B == 0:
            return out
        ws = MethodWorkspace(B, H, W, connectivity, "uf", device=image.device)
        _check(_lib.ccl_label_equal_async(
            ctypes.c_void_p(image.data_ptr()), B, H, W, int(connectivity), ctypes.c_void_p(out.data_ptr()),
            ws.ptr(), ws.nbytes, _stream_ptr(s)), "ccl_label_equal_async")
    return out


def label_3d(volume, connectivity: int = 26, *, out=None, stream=None):
    """3D volumes (NEXT-4, ccl_label_3d_async): uint8 CUDA [D,H,W] or
    [B,D,H,W], 6- or 26-connectivity -> int32 labels (0 or 1 + minimum raster
    index (z*H + y)*W + x of the component)."""
    torch = _torch()
    _check_image(volume)
    if volume.dim() == 3:
        B, (D, H, W) = 1, volume.shape
    elif volume.dim() == 4:
        B, D, H, W = volume.shape
    else:
        raise ValueError("expected [D,H,W] or [B,D,H,W]")
    with _on(volume.device, stream) as s:
        if out is None:
            out = torch.empty(volume.shape, dtype=torch.int32, device=volume.device)
        else:
            _check_out(out, volume.shape, volume.device)
        if B == 0:
            return out
        n = int(_lib.ccl_workspace_bytes_3d(B, D, H, W, int(connectivity)))
        ws = torch.empty(max(n, 1), dtype=torch.uint8, device=volume.device)
        _check(_lib.ccl_label_3d_async(
            ctypes.c_void_p(volume.data_ptr()), B, D, H, W, int(connectivity), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(ws.data_ptr()), n, _stream_ptr(s)), "ccl_label_3d_async")
    return out


STATS_FIELDS = ("label", "area", "x_min", "y_min", "x_max", "y_max", "sum_x", "sum_y")


def component_stats(labels, max_components: int | None = None, stream=None, relabel: bool = False):
    """Per-component statistics of a label map from label() (NEXT-3,
    ccl_component_stats_relabel_async): returns (counts [B] int32, dict field
    -> tensor [B, max_components]) with the components of each image in
    increasing label order (record k = component k+1 of the 1..K numbering).
    Records beyond counts[b] (or beyond max_components) are not written.
    relabel=True also returns the compacted label map (1..K per image, 0 =
    background) as a third element."""
    torch = _torch()
    if not isinstance(labels, torch.Tensor) or not labels.is_cuda or labels.dtype != torch.int32:
        raise TypeError("labels must be a CUDA int32 tensor")
    if not labels.is_contiguous():
        raise ValueError("labels must be contiguous")
    B, H, W = _shape3(labels)
    if max_components is None:
        max_components = (H * W + 1) // 2 + 1  # 4-conn checkerboard bound
    with _on(labels.device, stream) as s:
        rec = torch.empty((max(B, 1), max_components, 40), dtype=torch.uint8, device=labels.device)
        counts = torch.zeros(max(B, 1), dtype=torch.int32, device=labels.device)
        ws_n = int(_lib.ccl_stats_workspace_bytes(B, H, W))
        ws = torch.empty(max(ws_n, 1), dtype=torch.uint8, device=labels.device)
        rl = torch.empty(labels.shape, dtype=torch.int32, device=labels.device) if relabel else None
        _check(_lib.ccl_component_stats_relabel_async(
            ctypes.c_void_p(labels.data_ptr()), B, H, W, int(max_components), ctypes.c_void_p(rec.data_ptr()),
            ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(rl.data_ptr() if relabel else 0),
            ctypes.c_void_p(ws.data_ptr()), ws_n, _stream_ptr(s)),
            "ccl_component_stats_relabel_async")
    i32 = rec.view(torch.int32)  # [B, max, 10]
    i64 = rec.view(torch.int64)  # [B, max, 5]
    out = {f: i32[..., k] for k, f in enumerate(STATS_FIELDS[:6])}
    out["sum_x"] = i64[..., 3]
    out["sum_y"] = i64[..., 4]
    if relabel:
        return counts[:B], {k: v[:B] for k, v in out.items()}, rl
    return counts[:B], {k: v[:B] for k, v in out.items()}


def stages(image, connectivity: int, out, workspace: Workspace, tile_rows: int = 0, stream=None):
    """Enqueue K1, K2, K3 as three separate C-ABI calls (per-kernel timing)."""
    B, H, W = _shape3(image)
    _same_device(image.device, out, workspace.buf)
    s = _stream_ptr(stream)
    ws = workspace.ptr()
    _check(_lib.ccl_stage_local_merge(ctypes.c_void_p(image.data_ptr()), B, H, W, connectivity, ws,
                                      workspace.nbytes, tile_rows, s), "ccl_stage_local_merge")
    _check(_lib.ccl_stage_boundary(B, H, W, connectivity, ws, workspace.nbytes, tile_rows, s),
           "ccl_stage_boundary")
    _check(_lib.ccl_stage_link(B, H, W, connectivity, ctypes.c_void_p(out.data_ptr()), ws,
                               workspace.nbytes, tile_rows, s), "ccl_stage_link")


def stage_fns():
    """(k1, k2, k3) callables taking (image, connectivity, out, workspace,
    tile_rows, stream) for per-kernel event timing."""
    def k1(image, conn, out, ws, tile_rows=0, stream=None):
        B, H, W = _shape3(image)
        _check(_lib.ccl_stage_local_merge(ctypes.c_void_p(image.data_ptr()), B, H, W, conn, ws.ptr(),
                                          ws.nbytes, tile_rows, _stream_ptr(stream)), "k1")

    def k2(image, conn, out, ws, tile_rows=0, stream=None):
        B, H, W = _shape3(image)
        _check(_lib.ccl_stage_boundary(B, H, W, conn, ws.ptr(), ws.nbytes, tile_rows,
                                       _stream_ptr(stream)), "k2")

    def k3(image, conn, out, ws, tile_rows=0, stream=None):
        B, H, W = _shape3(image)
        _check(_lib.ccl_stage_link(B, H, W, conn, ctypes.c_void_p(out.data_ptr()), ws.ptr(),
                                   ws.nbytes, tile_rows, _stream_ptr(stream)), "k3")
    return k1, k2, k3


class HostSession:
    """End-to-end use from host memory: pinned host buffers + device scratch;
    ``run()`` enqueues H2D copy, the three kernels and the D2H copy through the
    C ABI (ccl_label_host_async) and synchronises."""

    def __init__(self, B: int, H: int, W: int, connectivity: int = 8):
        torch = _torch()
        self.B, self.H, self.W, self.conn = B, H, W, connectivity
        n = int(_lib.ccl_host_scratch_bytes(B, H, W, connectivity))
        if n == 0:
            raise ValueError("invalid geometry")
        self.scratch_bytes = n
        self.scratch = torch.empty(n, dtype=torch.uint8, device="cuda")
        self.h_image = torch.empty((B, H, W), dtype=torch.uint8, pin_memory=True)
        self.h_labels = torch.empty((B, H, W), dtype=torch.int32, pin_memory=True)

    def run(self, stream=None):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(_lib.ccl_label_host_async(
            ctypes.c_void_p(self.h_image.data_ptr()), self.B, self.H, self.W, self.conn,
            ctypes.c_void_p(self.h_labels.data_ptr()), ctypes.c_void_p(self.scratch.data_ptr()),
            self.scratch_bytes, ctypes.c_void_p(s.cuda_stream)), "ccl_label_host_async")
        s.synchronize()
        return self.h_labels

    @property
    def h2d_bytes(self):
        return self.B * self.H * self.W

    @property
    def d2h_bytes(self):
        return 4 * self.B * self.H * self.W


class HostPipeline:
    """End-to-end labeling of a stream of host images: ``depth`` HostSessions
    (pinned host buffers + device scratch) on ``depth`` CUDA streams, used
    round-robin, so that step i's device->host copy of its labels overlaps
    step i+1's host->device copy and kernels (PCIe is full duplex).  Every
    step still copies its own image in and its own labels out through
    ccl_label_host_async."""

    def __init__(self, B: int, H: int, W: int, connectivity: int = 8, depth: int = 2):
        torch = _torch()
        self.sessions = [HostSession(B, H, W, connectivity) for _ in range(depth)]
        self.streams = [torch.cuda.Stream() for _ in range(depth)]

    def enqueue(self, i: int):
        """Enqueue step i (no synchronisation); returns its session."""
        sess, st = self.sessions[i % len(self.sessions)], self.streams[i % len(self.streams)]
        _check(_lib.ccl_label_host_async(
            ctypes.c_void_p(sess.h_image.data_ptr()), sess.B, sess.H, sess.W, sess.conn,
            ctypes.c_void_p(sess.h_labels.data_ptr()), ctypes.c_void_p(sess.scratch.data_ptr()),
            sess.scratch_bytes, ctypes.c_void_p(st.cuda_stream)), "ccl_label_host_async")
        return sess


# ------------------------------------------------------------- strip sharding
class StripLabeler:
    """Row-strip sharded labeling of one H_total x W image: this object owns
    the per-rank buffers; ``local`` -> (caller all-gathers ``send``) ->
    ``finalize``.  ``label`` does all three with torch.distributed."""

    def __init__(self, rows: int, W: int, row0: int, H_total: int, k: int, rank: int,
                 connectivity: int = 8, device=None):
        torch = _torch()
        self.rows, self.W, self.row0, self.H, self.k, self.rank, self.conn = rows, W, row0, H_total, k, rank, connectivity
        n = int(_lib.ccl_strip_workspace_bytes(rows, W, k, connectivity))
        if n == 0:
            raise ValueError("invalid strip geometry")
        dev = device or "cuda"
        self.ws_bytes = n
        self.ws = torch.empty(n, dtype=torch.uint8, device=dev)
        self.send = torch.empty(4 * W, dtype=torch.int32, device=dev)
        self.gathered = torch.empty(k * 4 * W, dtype=torch.int32, device=dev)
        self.out = torch.empty((rows, W), dtype=torch.int32, device=dev)

    def local(self, strip, stream=None):
        _check_image(strip)
        _same_device(self.ws.device, strip)
        with _on(self.ws.device, stream) as s:
            _check(_lib.ccl_strip_local(ctypes.c_void_p(strip.data_ptr()), self.rows, self.W, self.row0, self.H,
                                        self.conn, self.k, ctypes.c_void_p(self.send.data_ptr()),
                                        ctypes.c_void_p(self.out.data_ptr()), ctypes.c_void_p(self.ws.data_ptr()),
                                        self.ws_bytes, _stream_ptr(s)), "ccl_strip_local")
        return self.send

    def finalize(self, gathered=None, stream=None):
        g = self.gathered if gathered is None else gathered
        _same_device(self.ws.device, g)
        with _on(self.ws.device, stream) as s:
            _check(_lib.ccl_strip_finalize(ctypes.c_void_p(g.data_ptr()), self.k, self.rank, self.rows, self.W,
                                           self.row0, self.H, self.conn, ctypes.c_void_p(self.out.data_ptr()),
                                           ctypes.c_void_p(self.ws.data_ptr()), self.ws_bytes, _stream_ptr(s)),
                   "ccl_strip_finalize")
        return self.out

    def label(self, strip, group=None):
        """local -> NCCL all-gather of the 4W-int edge buffers -> finalize."""
        import torch.distributed as dist
        self.local(strip)
        dist.all_gather_into_tensor(self.gathered, self.send, group=group)
        return self.finalize()


def strip_bounds(H: int, k: int, r: int):
    """Rows [row0, row1) of strip r when H rows are split into k contiguous
    strips as evenly as possible (the first H % k strips get one extra row)."""
    base, extra = divmod(H, k)
    row0 = r * base + min(r, extra)
    return row0, row0 + base + (1 if r < extra else 0)


def label_strips_emulated(image, k: int, connectivity: int = 8):
    """Single-GPU emulation of k-way strip sharding (the all-gather becomes a
    device copy): runs every rank's local and finalize stages on this GPU and
    returns the assembled [H, W] labels (tests / smoke)."""
    torch = _torch()
    _check_image(image)
    H, W = int(image.shape[0]), int(image.shape[1])
    if not 1 <= k <= H:
        raise ValueError("need 1 <= k <= H")
    labelers = []
    for r in range(k):
        r0, r1 = strip_bounds(H, k, r)
        lab = StripLabeler(r1 - r0, W, r0, H, k, r, connectivity, device=image.device)
        lab.local(image[r0:r1])
        labelers.append(lab)
    gathered = torch.cat([lab.send for lab in labelers])
    return torch.cat([lab.finalize(gathered) for lab in labelers])

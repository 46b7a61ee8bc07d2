"""C-ABI boundary tests that need no GPU: the library loads, exports every
symbol include/ccl.h declares, and rejects bad arguments with the documented
status codes BEFORE touching the device; host-side launch bookkeeping."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ccl.h")


@pytest.fixture(scope="module")
def ccl():
    import __graft_entry__
    __graft_entry__._load_build_module().build()
    import paper_1708_08180_b200 as m
    return m


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ccl_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = header_functions()
    for must in ("ccl_label", "ccl_label_batched", "ccl_label_batched_async", "ccl_workspace_bytes",
                 "ccl_stage_local_merge", "ccl_stage_boundary", "ccl_stage_link", "ccl_label_host_async"):
        assert must in names


def test_every_header_symbol_is_exported_and_bound(ccl):
    lib = ctypes.CDLL(ccl.LIB_PATH)
    for name in header_functions():
        assert hasattr(lib, name), f"libccl.so does not export {name}"
        assert name in ccl.SIGNATURES, f"binding lacks {name}"


def test_nm_exports_are_unmangled(ccl):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", ccl.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ccl_[a-z0-9_]+)\b", out))
    assert set(header_functions()) <= exported


FAKE_A = ctypes.c_void_p(0x10000000)
FAKE_B = ctypes.c_void_p(0x20000000)
FAKE_WS = ctypes.c_void_p(0x30000000)


def test_validation_codes(ccl):
    L = ccl.raw()
    conn = 8
    # null pointers
    assert L.ccl_label(None, 4, 4, conn, FAKE_B) == 1
    assert L.ccl_label(FAKE_A, 4, 4, conn, None) == 1
    # dimensions
    assert L.ccl_label(FAKE_A, 0, 4, conn, FAKE_B) == 2
    assert L.ccl_label(FAKE_A, 4, 0, conn, FAKE_B) == 2
    assert L.ccl_label_batched(FAKE_A, -1, 4, 4, conn, FAKE_B) == 2
    # too large: H*W > 2^31-1
    assert L.ccl_label(FAKE_A, 65536, 32769, conn, FAKE_B) == 3
    assert L.ccl_label(FAKE_A, 1, (1 << 31), conn, FAKE_B) == 3
    # connectivity
    for bad in (0, 1, 6, 9):
        assert L.ccl_label(FAKE_A, 4, 4, bad, FAKE_B) == 4
    # aliasing image/labels
    assert L.ccl_label(FAKE_A, 4, 4, conn, ctypes.c_void_p(0x10000004)) == 5
    # workspace too small
    need = ccl.workspace_bytes(1, 64, 64, conn)
    assert L.ccl_label_batched_async(FAKE_A, 1, 64, 64, conn, FAKE_B, FAKE_WS, need - 1, None) == 6
    # workspace overlapping the image
    assert L.ccl_label_batched_async(FAKE_A, 1, 64, 64, conn, FAKE_B, ctypes.c_void_p(0x10000000 - 256),
                                     need, None) == 5
    # workspace not 256-byte aligned (include/ccl.h; the kernels use 16-byte vector accesses)
    for off in (4, 8, 16, 128):
        assert L.ccl_label_batched_async(FAKE_A, 1, 64, 64, conn, FAKE_B, ctypes.c_void_p(0x30000000 + off),
                                         need, None) == 6
    # unsupported tile config
    assert L.ccl_label_batched_cfg_async(FAKE_A, 1, 64, 64, conn, FAKE_B, FAKE_WS, need, 7, None) == 8
    # B == 0 is a no-op
    assert L.ccl_label_batched(None, 0, 4, 4, conn, None) == 0
    assert L.ccl_label_batched_async(None, 0, 4, 4, conn, None, None, 0, None) == 0
    # status strings
    for code in range(9):
        assert ccl.status_string(code)
    assert "connectivity" in ccl.status_string(4)


def test_workspace_bytes(ccl):
    assert ccl.workspace_bytes(1, 0, 4, 8) == 0
    assert ccl.workspace_bytes(1, 4, 4, 5) == 0
    H, W = 1080, 1920
    n = ccl.workspace_bytes(3, H, W, 8)
    # bit mask (one uint32 word per 32 px per row) + run records (4 B per run,
    # worst case 512 runs per 1024-px tile row, rows rounded up to 32)
    bits = 3 * H * ((W + 31) // 32) * 4
    records = 3 * ((W + 1023) // 1024) * ((H + 31) // 32 * 32) * 512 * 4
    assert n >= bits + records
    # compact: edge slots instead of a per-pixel parent array
    assert n < 4.5 * 3 * H * W
    assert n % 256 == 0
    # the strip stages add the strip marks and the boundary slot union-find
    assert ccl.strip_workspace_bytes(H, W, 2, 8) > ccl.workspace_bytes(1, H, W, 8)


def boundaries(n, t):
    """Tile boundaries strictly inside [0, n): {k : k % t == 0, 0 < k < n}
    (reading R9 of DESIGN.md; brute-force enumeration)."""
    return [k for k in range(1, n) if k % t == 0]


def eq12(N, M, bx, by):
    """Eq. (1)-(2): P_x = floor(N/bx)*M, P_y = floor(M/by)*N."""
    return (N // bx) * M, (M // by) * N


def test_eq12_paper_numbers():
    # (4096, 4096, 32, 16) -> (524288, 1048576), launch max = 1048576
    px, py = eq12(4096, 4096, 32, 16)
    assert (px, py) == (524288, 1048576) and max(px, py) == 1048576


@pytest.mark.parametrize("H,W,ty", [(8192, 8192, 16), (4096, 4096, 8), (1080, 1920, 16), (33, 2049, 8),
                                    (1, 1, 16), (16, 1024, 16), (17, 1025, 32), (32768, 2048, 32)])
def test_boundary_work_items(ccl, H, W, ty):
    h, v = ccl.boundary_work_items(1, H, W, ty)
    tiles_x = -(-W // 1024)
    # horizontal: one warp per (interior row boundary, tile column); vertical:
    # one thread per (row, interior column boundary) -- brute-force enumeration
    assert h == len(boundaries(H, ty)) * tiles_x
    assert v == len(boundaries(W, 1024)) * H
    if H % ty == 0 and W % 1024 == 0:
        # Eq. (1)-(2) with (b_x, b_y) = (1024, ty) counts the x = 0 / y = 0 lines
        # too; the interior boundary cells are P_x - M and P_y - N.
        px, py = eq12(W, H, 1024, ty)
        assert v == px - H
        assert h * 1024 == py - W
    h3, v3 = ccl.boundary_work_items(3, H, W, ty)
    assert (h3, v3) == (3 * h, 3 * v)


def test_boundary_enumeration_covers_non_multiple_sizes():
    # the paper's printed id->cell map misses the last
    # boundary when the tile does not divide the size; our enumeration must not.
    assert boundaries(1080, 16)[-1] == 1072
    assert boundaries(10, 3) == [3, 6, 9]
    assert boundaries(33, 32) == [32]


def test_import_fails_loudly_without_library(tmp_path):
    # the binding refuses to import when libccl.so is absent (no CPU fallback)
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_1708_08180_b200"
    shutil.copytree(os.path.join(ROOT, "paper_1708_08180_b200"), pkg,
                    ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_1708_08180_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "missing" in r.stderr


def test_strip_validation(ccl):
    L = ccl.raw()
    need = L.ccl_strip_workspace_bytes(64, 1024, 4, 8)
    assert need > ccl.workspace_bytes(1, 64, 1024, 8)
    assert L.ccl_strip_workspace_bytes(64, 1024, 0, 8) == 0
    # rank / k / row0 out of range
    assert L.ccl_strip_finalize(FAKE_A, 4, 4, 64, 1024, 0, 256, 8, FAKE_B, FAKE_WS, need, None) == 2
    assert L.ccl_strip_local(FAKE_A, 64, 1024, 200, 256, 8, 4, FAKE_B, ctypes.c_void_p(0x40000000),
                             FAKE_WS, need, None) == 2
    # global labels must fit int32
    assert L.ccl_strip_local(FAKE_A, 64, 65536, 0, 40000, 8, 4, FAKE_B, ctypes.c_void_p(0x40000000),
                             FAKE_WS, need, None) == 3
    # workspace too small
    assert L.ccl_strip_local(FAKE_A, 64, 1024, 0, 256, 8, 4, FAKE_B, ctypes.c_void_p(0x40000000),
                             FAKE_WS, need - 1, None) == 6


def test_strip_bounds_partition(ccl):
    for H in (1, 7, 8, 100, 1080, 32768):
        for k in (1, 2, 3, 4, 8):
            if k > H:
                continue
            spans = [ccl.strip_bounds(H, k, r) for r in range(k)]
            assert spans[0][0] == 0 and spans[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_default_tile_rows(ccl):
    """The tile_rows = 0 rule: one of 8 / 16 / 32, never shorter for more work."""
    prev = 0
    for H in (16, 512, 2048, 8192, 32768):
        ty = ccl.default_tile_rows(1, H, 8192)
        assert ty in (8, 16, 32)
        assert ty >= prev
        prev = ty
    with pytest.raises(ValueError):
        ccl.default_tile_rows(1, 0, 5)

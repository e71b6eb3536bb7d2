"""CPU-side checks of the C-ABI boundary: libsattn.so loads, exports every function
include/sattn.h declares, and its synchronous argument validation rejects bad
descriptors before anything touches the GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sattn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"^typedef[^;]*;", "", src, flags=re.M | re.S)
    names = re.findall(r"^[A-Za-z_][\w\s\*]*?\b(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "defined")))


@pytest.fixture(scope="module")
def lib():
    import paper_2302_13451_b200 as pkg
    if not os.path.exists(pkg.LIB_PATH):
        from paper_2302_13451_b200 import _build
        _build.build(verbose=False)
    return pkg.lib()


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("sa_forward", "sa_backward", "llsa_forward", "llsa_backward", "sattn_stack_forward",
              "sattn_stack_backward", "llsa_stream_step", "sattn_last_error"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    import paper_2302_13451_b200 as pkg
    from paper_2302_13451_b200 import dist
    for n in _declared():
        assert hasattr(lib, n), n
        assert n in pkg.EXPORTS or n in dist.EXPORTS, f"binding does not type {n}"


def test_desc_layout_matches_header():
    import paper_2302_13451_b200 as pkg
    # 4 x int64 + 6 x 32-bit fields, no padding
    assert ctypes.sizeof(pkg.Desc) == 56


def _desc(**kw):
    import paper_2302_13451_b200 as pkg
    base = dict(B=1, H=1, T=16, D=4, L=3, R=1, dtype=pkg.F32)
    base.update(kw)
    return pkg.make_desc(**base)


@pytest.mark.parametrize("kw,status", [
    (dict(T=0), 1), (dict(B=-1), 1), (dict(L=-1), 1), (dict(R=-2), 1),
    (dict(dtype=7), 1), (dict(D=3), 4), (dict(D=256), 4), (dict(B=300, H=300), 4),
])
def test_validation_rejects_bad_descriptors(lib, kw, status):
    d = _desc(**kw)
    p = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    st = lib.sa_forward(ctypes.byref(d), p, p, p, p, p, None)
    assert st == status
    assert lib.sattn_last_error()


def test_null_and_misaligned_pointers_rejected(lib):
    d = _desc()
    p = ctypes.c_void_p(16)
    assert lib.sa_forward(ctypes.byref(d), None, p, p, p, p, None) == 1
    assert lib.llsa_forward(ctypes.byref(d), ctypes.c_void_p(18), p, p, p, p, None) == 1


def test_workspace_and_saved_sizes(lib):
    import paper_2302_13451_b200 as pkg
    d = _desc(B=2, H=3, T=37, D=8, L=5, R=2)
    # delta + LSE*log2(e) (+ LLSA: staircase part of delta) per channel, rows padded to 40 frames
    assert lib.sa_backward_workspace(ctypes.byref(d)) == 2 * 2 * 3 * 40 * 4
    assert lib.llsa_backward_workspace(ctypes.byref(d)) == 3 * 3 * 2 * 3 * 40 * 4
    assert lib.sattn_stack_saved_bytes(ctypes.byref(d), pkg.MODE_SA, 2) > 0
    assert lib.sattn_stack_saved_bytes(ctypes.byref(d), 9, 2) == 0
    # bf16, D = 64 (tensor-core backward): the same padded rows
    tcd = _desc(B=1, H=1, T=37, D=64, L=5, R=2, dtype=pkg.BF16)
    assert lib.sa_backward_workspace(ctypes.byref(tcd)) == 2 * 1 * 40 * 4
    bad = _desc(T=0)
    assert lib.sa_backward_workspace(ctypes.byref(bad)) == 0


def test_stream_state_errors(lib):
    h = ctypes.c_void_p()
    assert lib.llsa_stream_create(ctypes.byref(_desc()), 0, ctypes.byref(h)) == 1
    assert lib.llsa_stream_step(None, None, None, None, None) == 1


def test_stored_band_abi(lib):
    # NEXT-4 entry points: row stride = W rounded up to 8 elements (G29); workspace = delta rows;
    # synchronous validation before anything is enqueued (no GPU needed)
    import paper_2302_13451_b200 as pkg
    for L, R, ld in ((5, 2, 8), (32, 8, 48), (0, 0, 8), (32, 16, 56), (7, 0, 8), (8, 0, 16)):
        d = _desc(B=2, H=3, T=37, D=8, L=L, R=R)
        assert lib.sa_p_ld(ctypes.byref(d)) == ld
    d = _desc(B=2, H=3, T=37, D=8, L=5, R=2)
    assert lib.sa_backward_p_workspace(ctypes.byref(d)) == 2 * 3 * 40 * 4
    bad = _desc(T=0)
    assert lib.sa_p_ld(ctypes.byref(bad)) == 0 and lib.sa_backward_p_workspace(ctypes.byref(bad)) == 0
    p = ctypes.c_void_p(16)
    assert lib.sa_forward_p(ctypes.byref(d), p, p, p, p, p, None, None) == 1          # NULL band
    assert lib.sa_forward_p(ctypes.byref(d), p, p, p, p, p, ctypes.c_void_p(18), None) == 1   # misaligned
    ws = 2 * 3 * 40 * 4
    assert lib.sa_backward_p(ctypes.byref(d), p, p, p, p, None, p, p, p, p, p, ws, None) == 1
    assert lib.sa_backward_p(ctypes.byref(d), p, p, p, p, p, p, p, p, p, p, ws - 4, None) == 3   # ECONFIG
    # impl = TC outside the tensor-core limits (fp32) -> EUNSUPPORTED before any launch
    t = _desc(B=1, H=1, T=16, D=64, L=3, R=1, impl="tc")
    assert lib.sa_forward_p(ctypes.byref(t), p, p, p, p, p, p, None) == 4
    tw = _desc(B=1, H=1, T=16, D=64, L=40, R=40, dtype=pkg.BF16, impl="tc")
    assert lib.sa_forward_p(ctypes.byref(tw), p, p, p, p, p, p, None) == 4
    assert lib.sattn_last_error()

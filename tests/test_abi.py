"""Host-side checks of the C ABI (no GPU needed): the library loads, exports every
symbol include/spion.h declares, and rejects bad arguments before launching anything."""
import ctypes
import os
import re

import pytest

from paper_2309_12578_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "spion.h")).read()
    return sorted(set(re.findall(r"SPION_API\s+[\w\s\*]+?\b(spion_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = _declared()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTS), "ctypes table out of sync with include/spion.h"


def test_no_oracle_in_product_package():
    pkg = os.path.join(ROOT, "paper_2309_12578_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "spion_oracle" not in txt, f


def test_sizes():
    lib = N.lib()
    assert lib.spion_bsr_plan_bytes(4096, 64) > 0
    assert lib.spion_bsr_plan_bytes(100, 64) == 0
    assert lib.spion_pattern_workspace_bytes(4096, 64) >= 64 * 64 * 8
    assert lib.spion_attn_workspace_bytes(128, 4096, 64, N.BF16) >= 128 * 4096 * 4  # D = rowsum(dO*O), fp32
    assert lib.spion_step_arena_bytes(2, 64, 16, 8, N.F32) > 0


def _bsr_dummy(L, B):
    s = N.BSR()
    fake = 256  # never dereferenced: validation fails first
    s.brow_ptr = s.bcol_idx = s.bcol_ptr = s.brow_idx = s.nnzb = fake
    s.nnzb_cap = (L // B) ** 2
    return s


@pytest.mark.parametrize("L,B,F,theta,kind,want", [
    (100, 64, 31, 90.0, 0, 1),      # L % B -> shape
    (0, 8, 31, 90.0, 0, 1),
    (64, 8, 30, 90.0, 0, 2),        # even filter -> param
    (64, 8, 31, 100.0, 0, 2),       # alpha outside (0,100)
    (64, 8, 31, 0.0, 1, 2),
    (64, 8, 31, float("nan"), 2, 2),
    (64, 8, 31, 90.0, 9, 2),        # bad enum
    (64 * 256, 8, 31, 90.0, 0, 7),  # nblk > 128 -> unsupported
])
def test_pattern_rejects_bad_arguments(L, B, F, theta, kind, want):
    lib = N.lib()
    s = _bsr_dummy(max(L, 1), B)
    st = lib.spion_pattern(ctypes.c_void_p(256), L, B, F, theta, kind, ctypes.c_void_p(256), 1 << 30,
                           ctypes.byref(s), None, None)
    assert st == want


def test_pattern_rejects_misaligned_and_small_workspace():
    lib = N.lib()
    s = _bsr_dummy(64, 8)
    assert lib.spion_pattern(ctypes.c_void_p(258), 64, 8, 31, 90.0, 0, ctypes.c_void_p(256), 1 << 30,
                             ctypes.byref(s), None, None) == 4
    assert lib.spion_pattern(ctypes.c_void_p(256), 64, 8, 31, 90.0, 0, ctypes.c_void_p(256), 8,
                             ctypes.byref(s), None, None) == 5


def test_attention_rejects_bad_arguments():
    lib = N.lib()
    s = _bsr_dummy(64, 8)
    s.L, s.block, s.nblk = 64, 8, 8
    P = ctypes.c_void_p(256)
    # d > 128
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 64, 256, 64 * 256, 256, N.F32, ctypes.byref(s), 0, 1.0, P, 256, None) == 1
    # pattern for another L
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 128, 16, 128 * 16, 16, N.F32, ctypes.byref(s), 0, 1.0, P, 256, None) == 1
    # bad mode / dtype
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 64, 16, 64 * 16, 16, N.F32, ctypes.byref(s), 5, 1.0, P, 256, None) == 2
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 64, 16, 64 * 16, 16, 7, ctypes.byref(s), 0, 1.0, P, 256, None) == 2
    # misaligned stride for bf16
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 64, 16, 64 * 20, 20, N.BF16, ctypes.byref(s), 0, 1.0, P, 256, None) == 4
    # workspace too small (forward: the 256-byte counter area; backward: counters + D + -lse*log2e)
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 64, 16, 64 * 16, 16, N.F32, ctypes.byref(s), 0, 1.0, P, 16,
                              None) == 5
    assert lib.spion_attn_fwd(P, P, P, P, P, 1, 64, 16, 64 * 16, 16, N.F32, ctypes.byref(s), 0, 1.0, None, 256,
                              None) == 2
    assert lib.spion_attn_bwd(P, P, P, P, P, P, P, P, P, 1, 64, 16, 64 * 16, 16, N.F32, ctypes.byref(s), 0, 1.0,
                              P, 16, None) == 5


def test_attn_path_query():
    """spion_attn_path is host-only: which kernel family a call would run, or -status."""
    lib = N.lib()
    s = _bsr_dummy(64, 8)
    s.L, s.block, s.nblk = 64, 8, 8
    assert lib.spion_attn_path(1, 64, 16, 64 * 16, 16, N.F32, ctypes.byref(s)) == N.PATH_CUDA_CORE
    assert lib.spion_attn_path(1, 64, 256, 64 * 256, 256, N.F32, ctypes.byref(s)) == -1   # d > 128: shape
    assert lib.spion_attn_path(1, 64, 16, 64 * 20, 20, N.BF16, ctypes.byref(s)) == -4     # stride % 8: align
    t = _bsr_dummy(4096, 64)
    t.L, t.block, t.nblk = 4096, 64, 64
    # bf16 d=64 B=64 without a plan cannot take the tensor-core path
    assert lib.spion_attn_path(128, 4096, 64, 4096 * 64, 64, N.BF16, ctypes.byref(t)) == N.PATH_CUDA_CORE
    t.plan, t.plan_bytes = 256, lib.spion_bsr_plan_bytes(4096, 64)
    # with a plan: tcgen05 where the driver entry point exists (GPU box), else the CUDA-core path
    assert lib.spion_attn_path(128, 4096, 64, 4096 * 64, 64, N.BF16, ctypes.byref(t)) in (N.PATH_CUDA_CORE,
                                                                                         N.PATH_TCGEN05)
    assert lib.spion_attn_fwd_workspace_bytes(128, 4096, 64, N.BF16) == 256
    # counters + D + -lse*log2e; for bf16 d=64 also the fused backward's completion counters (sized for
    # block 32) and fp32 dQ accumulator [bh][L][64]
    base = 256 + 2 * 128 * 4096 * 4
    assert lib.spion_attn_workspace_bytes(128, 4096, 32, N.BF16) == base
    assert lib.spion_attn_workspace_bytes(128, 4096, 64, N.F32) == base
    assert lib.spion_attn_workspace_bytes(128, 4096, 64, N.BF16) == base + 128 * 128 * 4 + 128 * 4096 * 64 * 4


def test_transition_rejects_bad_arguments():
    lib = N.lib()
    P = ctypes.c_void_p(256)
    assert lib.spion_transition(None, 0.1, P, None, None, None) == 2
    assert lib.spion_transition(P, 0.1, None, None, None, None) == 2
    assert lib.spion_transition(P, float("nan"), P, None, None, None) == 2
    assert lib.spion_transition(P, -1.0, P, None, None, None) == 2


def test_step_host_validates_before_copying():
    """Parameter errors come back before any copy is enqueued (the host pointers are bogus)."""
    lib = N.lib()
    P = ctypes.c_void_p(256)
    nb = lib.spion_step_arena_bytes(2, 64, 16, 8, N.F32)
    args = [P] * 10
    # even filter, alpha out of range, bad mode: all rejected synchronously, no CUDA call needed
    assert lib.spion_step_host(*args, 2, 64, 16, 8, 30, 75.0, 0, N.F32, 0, 0.25, P, nb, None, None) == 2
    assert lib.spion_step_host(*args, 2, 64, 16, 8, 31, 100.0, 0, N.F32, 0, 0.25, P, nb, None, None) == 2
    assert lib.spion_step_host(*args, 2, 64, 16, 8, 31, 75.0, 0, N.F32, 9, 0.25, P, nb, None, None) == 2
    assert lib.spion_step_host(*args, 2, 64, 256, 8, 31, 75.0, 0, N.F32, 0, 0.25, P,
                               lib.spion_step_arena_bytes(2, 64, 256, 8, N.F32), None, None) == 1


def test_status_strings():
    lib = N.lib()
    for k in range(8):
        assert lib.spion_status_str(k)


def test_pattern_pool_region_and_split_validation():
    """The multi-device pattern split (spion_pattern_pool / spion_pattern_finalize): the summable
    region of a pattern workspace (the int64 pool sums at byte 256 and the bad-score count at byte 8,
    contiguous) and the host-side rejections, all before any device work (bogus pointers)."""
    lib = N.lib()
    off = ctypes.c_size_t(7)
    for L, B in ((64, 8), (1024, 32), (4096, 64)):
        n = L // B
        cnt = lib.spion_pattern_pool_region(L, B, ctypes.byref(off))
        assert off.value == 8 and cnt == (256 - 8) // 8 + n * n
        assert off.value + 8 * cnt == lib.spion_pattern_workspace_bytes(L, B) - ((-(n * n * 8)) % 256)
    assert lib.spion_pattern_pool_region(100, 32, ctypes.byref(off)) == 0 and off.value == 0
    P = ctypes.c_void_p(1 << 20)  # 16-byte aligned bogus device pointer: never dereferenced
    ws = lib.spion_pattern_workspace_bytes(256, 16)
    # row range not at block boundaries / outside [0, L]
    assert lib.spion_pattern_pool(P, 256, 16, 31, 8, 40, P, ws, None) == 1
    assert lib.spion_pattern_pool(P, 256, 16, 31, 224, 288, P, ws, None) == 1
    assert lib.spion_pattern_pool(P, 256, 16, 31, 64, 32, P, ws, None) == 1
    # even filter, null workspace, misaligned scores, small workspace
    assert lib.spion_pattern_pool(P, 256, 16, 30, 0, 64, P, ws, None) == 2
    assert lib.spion_pattern_pool(P, 256, 16, 31, 0, 64, None, ws, None) == 2
    assert lib.spion_pattern_pool(ctypes.c_void_p((1 << 20) + 4), 256, 16, 31, 0, 64, P, ws, None) == 4
    assert lib.spion_pattern_pool(P, 256, 16, 31, 0, 64, P, ws - 1, None) == 5
    # finalize: alpha out of range, unknown variant bits, null output pattern
    assert lib.spion_pattern_finalize(256, 16, 100.0, N.THRESH["linear"], 0, P, ws, None, None, None) == 2
    assert lib.spion_pattern_finalize(256, 16, 50.0, N.THRESH["linear"], 8, P, ws, None, None, None) == 2
    assert lib.spion_pattern_finalize(256, 16, 50.0, N.THRESH["linear"], 0, P, ws, None, None, None) == 2

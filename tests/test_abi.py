"""CPU checks of the C ABI boundary: the library builds, loads, and exports every
symbol include/semipd.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import paper_2504_19867_b200 as spd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "semipd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(semipd_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = spd.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), f"missing export {s}"
    assert b"sm_100a" in L.semipd_version()


def test_host_only_calls():
    L = spd.lib()
    assert L.semipd_blocks_for_tokens(251, 16) == 16
    assert L.semipd_blocks_for_tokens(256, 16) == 16
    assert L.semipd_blocks_for_tokens(0, 16) == 0
    assert L.semipd_blocks_for_tokens(-1, 16) == -1
    cfg = spd.PoolConfig(2, 100, 16, 8, 128, 128, 4, 8).c(0)
    nb = L.semipd_kv_pool_bytes(ctypes.byref(cfg))
    kv = 2 * 100 * 8 * 16 * 128 * 2 * 2
    assert kv < nb < kv + 2 * 1024 * 1024
    bad = spd.PoolConfig(2, 100, 16, 8, 128, 128, 0, 8).c(0)
    assert L.semipd_kv_pool_bytes(ctypes.byref(bad)) == 0
    # NULL handle / arguments are rejected without touching a device
    assert L.semipd_set_partition(None, 50.0, 50.0) == spd.INVALID
    assert L.semipd_alloc_blocks(None, None, None, 1, None, None) == spd.INVALID
    assert L.semipd_kv_pool_create(ctypes.byref(cfg), None, 0, None, None) == spd.INVALID
    assert L.semipd_prefill_mla_expanded_workspace_bytes(None, 1, 100, 16) == 0
    assert L.semipd_prefill_mla_expanded(None, 0, None, None, None, None, None, None, None, 1, 1,
                                         1, 1, 16, 0.1, None, None, 0, 0, None, None) == spd.INVALID


def test_sass_is_blackwell_native():
    """The built library holds tcgen05 (UTCHMMA), TMEM (LDTM/STTM) and TMA (UTMALDG)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    sass = subprocess.run([tool, "-sass", spd.lib()._name], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "STTM", "UTMALDG"):
        assert mnem in sass, mnem


def test_peer_gather_host_argument_checks():
    """The peer-gather calls reject bad host arguments before touching a device."""
    L = spd.lib()
    vp = ctypes.c_void_p
    assert L.semipd_ipc_alloc(0, ctypes.byref(vp()), None) == spd.INVALID
    assert L.semipd_ipc_open(None, None) == spd.INVALID
    assert L.semipd_ipc_close(None) == spd.INVALID
    assert L.semipd_ipc_free(None) == spd.INVALID
    d = (vp * 2)(1, 2)
    f = (vp * 2)(3, 4)
    args = dict(src=vp(5), bytes=16, dsts=d, flags=f, mine=vp(6), world=2, rank=0)

    def call(**kw):
        a = {**args, **kw}
        return L.semipd_peer_gather(a["src"], a["bytes"], a["dsts"], a["flags"], a["mine"],
                                    a["world"], a["rank"], None)
    assert call(world=0) == spd.INVALID
    assert call(world=9) == spd.INVALID
    assert call(rank=2) == spd.INVALID
    assert call(mine=None) == spd.INVALID
    assert call(dsts=(vp * 2)(1, None)) == spd.INVALID
    assert call(src=None) == spd.INVALID


def test_fp8_pool_host_logic():
    """FP8 (E4M3) pools (reading R31): one byte per K / V element in the layout, and the FP8
    calls reject bad host arguments before touching a device."""
    import torch
    L = spd.lib()
    c8 = spd.PoolConfig(2, 100, 64, 8, 128, 128, 4, 8, dtype=torch.float8_e4m3fn).c(0)
    cb = spd.PoolConfig(2, 100, 64, 8, 128, 128, 4, 8).c(0)
    n8, nb = L.semipd_kv_pool_bytes(ctypes.byref(c8)), L.semipd_kv_pool_bytes(ctypes.byref(cb))
    kv8 = 2 * 100 * 8 * 64 * 128 * 2
    assert kv8 < n8 < kv8 + 2 * 1024 * 1024
    assert nb - n8 == kv8  # exactly half the bf16 pool's K / V bytes
    one = (ctypes.c_float * 2)(1.0, 1.0)
    assert L.semipd_set_kv_scales(None, one, one) == spd.INVALID
    assert L.semipd_fp8_prefill_scratch_bytes(None, 1) == 0
    assert L.semipd_set_fp8_prefill_scratch(None, None, 0, 1) == spd.INVALID

"""The C-ABI library loads without a GPU and exports every declared symbol;
NVRTC compiles sm_100a cubins on the CPU."""
import ctypes
import os
import re

from conftest import ROOT
from paper_2506_22609_b200 import native
from paper_2506_22609_b200.game import precompile


def declared():
    with open(os.path.join(ROOT, "include", "ludax_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(lx_\w+)\(", text, re.M)))


def test_every_header_symbol_is_exported():
    lib = native.lib()
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(native.EXPORTS)
    assert lib.lx_version() >= 100


def test_nvrtc_compiles_config_games_for_sm100a():
    keys = precompile(prune=False)
    for k in keys.values():
        for g in range(6):                     # one cubin per kernel group
            path = os.path.join(native.CACHE_DIR, f"{k}-g{g}.cubin")
            with open(path, "rb") as f:
                head = f.read(64)
            assert head[:4] == b"\x7fELF"


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        return
    h = ctypes.c_void_p()
    st = native.lib().lx_game_create(b"garbage", b"x", native.INCLUDE_DIR.encode(),
                                     b"", ctypes.byref(h))
    assert st == 4      # LX_ECOMPILE: the garbage never reaches the driver
    assert b"NVRTC" in native.lib().lx_last_error()


def test_host_buffer_calls_reject_bad_arguments_without_a_gpu():
    """lx_playout_host / _async / _wait validate their arguments before any
    driver call (LX_EINVALID = 6), so a bad binding fails cleanly."""
    L = native.lib()
    stuck = ctypes.c_int64(0)
    ticket = ctypes.c_int64(0)
    stats = (ctypes.c_uint64 * 8)()
    assert L.lx_playout_host(None, 16, 200, 0, 1, None, 0, None, None, stats, None,
                             ctypes.byref(stuck), None) == 6
    assert L.lx_playout_host_async(None, 16, 200, 0, 1, None, 0, None, None, stats, None,
                                   None, ctypes.byref(ticket)) == 6
    assert L.lx_playout_host_wait(None, 0, ctypes.byref(stuck)) == 6
    assert b"NULL" in L.lx_last_error()

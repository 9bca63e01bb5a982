"""Device binding of game handles (ludax_b200.cpp current_context / check_ctx):
a handle binds to the device whose context is current at create time; a
thread with no current context gets an error instead of a silent fallback to
device 0; lx_bind_device makes a device current for runtime-less callers;
lx_game_info reports the bound device."""
import ctypes
import threading

import pytest

from conftest import game_text

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import lowering, native, syntax  # noqa: E402


def _create(src):
    h = ctypes.c_void_p()
    st = native.lib().lx_game_create(src.encode(), b"c4", native.INCLUDE_DIR.encode(),
                                     native.CACHE_DIR.encode(), ctypes.byref(h))
    return st, h, native.lib().lx_last_error().decode()


def test_no_current_context_is_an_error_then_bind_device():
    src = lowering.lower_game(syntax.parse_game(game_text("connect_four"))).source
    out = {}

    def worker():                      # a fresh thread: no CUDA context is current
        out["first"] = _create(src)[::2]
        out["bind"] = native.lib().lx_bind_device(0)
        st, h, err = _create(src)
        info = native.GameInfo()
        native.lib().lx_game_info_get(h, ctypes.byref(info))
        out["second"] = (st, info.device, info.num_cells, info.state_quads)
        native.lib().lx_game_destroy(h)
    t = threading.Thread(target=worker)
    t.start()
    t.join()
    st, err = out["first"]
    assert st == 5 and "no current CUDA context" in err          # LX_ECUDA
    assert out["bind"] == 0
    assert out["second"][:3] == (0, 0, 42)
    assert native.lib().lx_bind_device(99) == 6                   # LX_EINVALID: no such device


def test_handle_reports_its_device_and_launches_there():
    torch.cuda.set_device(0)
    g = lx.load_config_game("connect_four")
    assert g.native.info.device == torch.cuda.current_device()
    st = g.init(64, seed=1)
    assert st.words.device.index == g.native.info.device
    final, stats = g.rollout(batch_size=64, seed=1)
    assert int(stats[5]) == 64

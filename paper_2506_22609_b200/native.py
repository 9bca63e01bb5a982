"""ctypes binding of libludax_b200.so (C-ABI: include/ludax_b200.h).

There is no fallback: if the library is missing or the CUDA driver is not
usable, calls raise.  ``build_native`` compiles the library in-tree; the
five config games' cubins are precompiled by ``precompile`` (NVRTC, sm_100a)
into ``csrc/_cubin`` so a GPU box only loads them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import raise_status

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_native", "libludax_b200.so")
INCLUDE_DIR = os.path.join(PKG, "csrc", "device")
CACHE_DIR = os.path.join(PKG, "csrc", "_cubin")


class GameInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in (
        "num_cells", "num_actions", "pass_index", "board_words", "state_quads", "state_bytes",
        "private_words", "mechanics", "mask_words", "device", "num_sms", "rollout_blocks",
        "rollout_threads")]


REF_FIELDS = ("board_piece", "board_owner", "current_player", "move_count", "terminated",
              "truncated", "outcome", "seeds", "scores", "pass_streak", "pass_flags",
              "last_mover", "last_kind", "last_source", "last_dest", "last_dest_by_player",
              "comp_labels", "phase", "must_move", "turn_pos", "hopped_mask", "captured_mask",
              "promoted_mask")


class RefState(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in REF_FIELDS]


EXPORTS = ("lx_version", "lx_last_error", "lx_game_create", "lx_bind_device", "lx_compile_only",
           "lx_cache_key", "lx_game_info_get", "lx_game_destroy", "lx_init", "lx_legal",
           "lx_sample", "lx_truncate", "lx_set_seeds", "lx_step", "lx_random_step", "lx_rollout",
           "lx_export", "lx_import", "lx_observe", "lx_env_step", "lx_expand", "lx_mcts",
           "lx_playout_host", "lx_playout_host_async", "lx_playout_host_wait")


def build_native():
    subprocess.run(["make", "-s", "-C", os.path.join(PKG, "csrc")], check=True)


_lib = None


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(make -C paper_2506_22609_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
    cs = ctypes.c_char_p
    L.lx_version.restype = i32
    L.lx_last_error.restype = cs
    L.lx_game_create.argtypes = [cs, cs, cs, cs, ctypes.POINTER(vp)]
    L.lx_compile_only.argtypes = [cs, cs, cs, cs, ctypes.c_char_p]
    L.lx_game_info_get.argtypes = [vp, ctypes.POINTER(GameInfo)]
    L.lx_cache_key.argtypes = [cs, cs, ctypes.c_char_p]
    L.lx_game_destroy.argtypes = [vp]
    L.lx_init.argtypes = [vp, vp, i64, vp, u64, i64, vp]
    L.lx_bind_device.argtypes = [i32]
    L.lx_legal.argtypes = [vp, vp, i64, vp, vp, vp, vp]
    L.lx_sample.argtypes = [vp, vp, i64, vp, vp, vp, vp]
    L.lx_truncate.argtypes = [vp, vp, i64, vp, vp]
    L.lx_set_seeds.argtypes = [vp, vp, i64, vp, vp]
    L.lx_step.argtypes = [vp, vp, i64, vp, vp, i32, vp, ctypes.POINTER(i64), vp]
    L.lx_random_step.argtypes = [vp, vp, i64, i32, vp, vp]
    L.lx_rollout.argtypes = [vp, vp, i64, i32, i32, u64, vp, i64, vp, vp, vp, vp, i32,
                             ctypes.POINTER(i64), vp]
    L.lx_playout_host.argtypes = [vp, i64, i32, i32, u64, vp, i64, vp, vp, vp, vp,
                                  ctypes.POINTER(i64), vp]
    L.lx_playout_host_async.argtypes = [vp, i64, i32, i32, u64, vp, i64, vp, vp, vp, vp, vp,
                                        ctypes.POINTER(i64)]
    L.lx_playout_host_wait.argtypes = [vp, i64, ctypes.POINTER(i64)]
    L.lx_expand.argtypes = [vp, vp, i64, vp, vp, vp, i64, vp, ctypes.c_int, vp, vp, vp, vp]
    L.lx_mcts.argtypes = [vp, vp, i64, vp, vp, ctypes.c_double, ctypes.c_int, vp, ctypes.c_int,
                          vp, i64, ctypes.c_int, vp, i64, vp, vp, ctypes.c_int, vp]
    L.lx_export.argtypes = [vp, vp, i64, ctypes.POINTER(RefState), vp]
    L.lx_import.argtypes = [vp, vp, i64, ctypes.POINTER(RefState), vp]
    L.lx_observe.argtypes = [vp, vp, i64, i32, vp, vp]
    L.lx_env_step.argtypes = [vp, vp, i64, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp]
    for name in EXPORTS:
        if name not in ("lx_version", "lx_last_error"):
            getattr(L, name).restype = i32
    _lib = L
    return L


def check(status, bad_row=-1):
    if status != 0:
        raise_status(status, lib().lx_last_error().decode(errors="replace"), bad_row)


def compile_only(source, name):
    key = ctypes.create_string_buffer(80)
    os.makedirs(CACHE_DIR, exist_ok=True)
    check(lib().lx_compile_only(source.encode(), name.encode(), INCLUDE_DIR.encode(),
                                CACHE_DIR.encode(), key))
    return key.value.decode()


def cache_key(source):
    key = ctypes.create_string_buffer(80)
    check(lib().lx_cache_key(source.encode(), INCLUDE_DIR.encode(), key))
    return key.value.decode()


class NativeGame:
    """Owns one lx_game handle (modules loaded on the current CUDA context,
    i.e. bound to the current device)."""

    def __init__(self, source, name, expect=None):
        h = ctypes.c_void_p()
        os.makedirs(CACHE_DIR, exist_ok=True)
        check(lib().lx_game_create(source.encode(), name.encode(), INCLUDE_DIR.encode(),
                                   CACHE_DIR.encode(), ctypes.byref(h)))
        self.h = h
        info = GameInfo()
        check(lib().lx_game_info_get(self.h, ctypes.byref(info)))
        self.info = info
        for k, v in (expect or {}).items():     # the lowering and the device unit agree
            if getattr(info, k) != v:
                raise RuntimeError(f"{name}: lx_game_info.{k} = {getattr(info, k)}, "
                                   f"lowering says {v}")

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.lx_game_destroy(self.h)
                self.h = None
        except Exception:
            pass

"""TEST INFRASTRUCTURE: compile a lowered game's rules for the host (g++)
and run playouts in the reference GameState layout (see hostsim.cpp)."""
import ctypes
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DEVICE = os.path.join(ROOT, "paper_2506_22609_b200", "csrc", "device")
BUILD = os.path.join(HERE, "build")

FIELDS = ("board_piece", "board_owner", "current_player", "move_count", "terminated",
          "truncated", "outcome", "seeds", "scores", "pass_streak", "pass_flags",
          "last_mover", "last_kind", "last_source", "last_dest", "last_dest_by_player",
          "comp_labels", "phase", "must_move", "turn_pos", "hopped_mask", "captured_mask",
          "promoted_mask")


class _Ref(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in FIELDS]


class HostGame:
    def __init__(self, lowered):
        src = lowered.source.replace('#include "lx_kernels.cuh"', "")
        hdrs = "".join(open(os.path.join(DEVICE, h)).read()
                       for h in ("lx_core.cuh", "lx_rules.cuh"))
        key = hashlib.sha256((src + hdrs + open(os.path.join(HERE, "hostsim.cpp")).read())
                             .encode()).hexdigest()[:20]
        os.makedirs(BUILD, exist_ok=True)
        gsrc = os.path.join(BUILD, f"{key}.h")
        so = os.path.join(BUILD, f"{key}.so")
        if not os.path.exists(so):
            with open(gsrc, "w") as f:
                f.write(src)
            subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-ffp-contract=off",
                            "-fno-gnu-unique", "-fvisibility=hidden", "-fvisibility-inlines-hidden",
                            "-w", f"-I{HERE}", f"-I{DEVICE}", f'-DGAME_SOURCE="{gsrc}"',
                            os.path.join(HERE, "hostsim.cpp"), "-o", so + ".tmp"], check=True)
            os.replace(so + ".tmp", so)
        self.lib = ctypes.CDLL(so)
        self.lib.sim_playout.restype = ctypes.c_int64
        self.lib.sim_playout.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.POINTER(_Ref)]
        self.lib.sim_transcript.restype = ctypes.c_int
        self.lib.sim_transcript.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.POINTER(_Ref)]
        self.lib.sim_masks.restype = ctypes.c_int
        self.lib.sim_masks.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p]
        self.info = lowered.info

    def layout(self):
        """(NWORDS, NQ) of the device state layout as lx::Layout computes it."""
        out = (ctypes.c_int * 2)()
        self.lib.sim_layout(out)
        return out[0], out[1]

    def playout(self, seeds, max_turns=200, layout_arrays=None):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        arrays = layout_arrays(len(seeds))
        ref = _Ref(**{f: (arrays[f].ctypes.data if f in arrays else None) for f in FIELDS})
        steps = self.lib.sim_playout(len(seeds), seeds.ctypes.data, max_turns, ctypes.byref(ref))
        arrays["seeds"][:] = seeds
        return arrays, steps

    def masks(self, seed, max_plies=400):
        A = self.info["A"]
        m = np.zeros((max_plies, A), np.uint8)
        a = np.zeros(max_plies, np.int64)
        t = self.lib.sim_masks(seed, max_plies, m.ctypes.data, a.ctypes.data)
        return m[:t].astype(bool), a[:t]

    def transcript(self, actions, seed=0, layout_arrays=None):
        """Apply scripted actions from init(batch_size=1, seed=seed) (the env
        seed is spawn_seeds(seed, 1)[0], reference compiler.py:357-364);
        returns (arrays, masks
        (n+1, A) before each ply and after the last, legal flags, plies)."""
        acts = np.ascontiguousarray(actions, dtype=np.int64)
        n = len(acts)
        A = self.info["A"]
        m = np.zeros((n + 1, A), np.uint8)
        ok = np.zeros(max(n, 1), np.uint8)
        arrays = layout_arrays(1)
        ref = _Ref(**{f: (arrays[f].ctypes.data if f in arrays else None) for f in FIELDS})
        from paper_2506_22609_b200 import rng
        env_seed = int(rng.spawn_seeds(seed, 1)[0])
        t = self.lib.sim_transcript(env_seed, n, acts.ctypes.data, m.ctypes.data, ok.ctypes.data,
                                    ctypes.byref(ref))
        return arrays, m.astype(bool), ok[:n].astype(bool), t

"""The C-ABI from C: tests/c_abi_smoke.c includes only include/ludax_b200.h,
sizes every buffer from lx_game_info, and drives bind -> create -> info ->
init -> rollout -> export.  CPU: it compiles against the header (gcc, C99,
-Wall -Werror).  GPU: it runs, and its exported final states equal the CPU
oracle's for the same seeds."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, game_text, has_gpu
from oracle import oracle as O
from paper_2506_22609_b200 import lowering, native, syntax

CUDA = "/usr/local/cuda"
SRC = os.path.join(ROOT, "tests", "c_abi_smoke.c")


def _build(tmp_path, link):
    exe = str(tmp_path / ("c_abi_smoke" if link else "c_abi_smoke.o"))
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O1", f"-I{ROOT}/include",
           f"-I{CUDA}/include", SRC]
    if link:
        cmd += ["-o", exe, f"-L{os.path.dirname(native.LIB_PATH)}", "-lludax_b200",
                f"-Wl,-rpath,{os.path.dirname(native.LIB_PATH)}", f"-L{CUDA}/lib64",
                "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
    else:
        cmd += ["-c", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_caller_compiles_against_header(tmp_path):
    _build(tmp_path, link=False)


def _read_dump(path):
    out = {}
    with open(path, "rb") as f:
        while True:
            name = f.readline().strip().decode()
            if not name:
                break
            n = int(np.frombuffer(f.read(8), np.uint64)[0])
            out[name] = f.read(n)
    return out


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name,B", [("connect_four", 4096), ("hex", 512), ("reversi", 1024),
                                    ("pente", 128), ("english_draughts", 256)])
def test_c_caller_rollout_matches_oracle(tmp_path, name, B):
    exe = _build(tmp_path, link=True)
    low = lowering.lower_game(syntax.parse_game(game_text(name)))
    src = tmp_path / f"{name}.cu"
    src.write_text(low.source)
    out = tmp_path / "out.bin"
    p = subprocess.run([exe, str(src), name, native.INCLUDE_DIR, native.CACHE_DIR, str(B), "77",
                        str(out)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    info = dict(kv.split("=") for kv in p.stdout.splitlines()[0].split()[1:])
    assert int(info["C"]) == low.info["C"] and int(info["A"]) == low.info["A"]
    assert int(info["pass"]) == low.info["pass_index"] and int(info["NQ"]) == low.info["nq"]
    assert int(info["W"]) == low.info["W"] and int(info["state_bytes"]) == 16 * low.info["nq"]
    got = _read_dump(out)
    want, steps = O.OracleGame(name).playout(B, seed=77)
    C = low.info["C"]
    for f, dt, shape in (("board_piece", np.int8, (B, C)), ("board_owner", np.int8, (B, C)),
                         ("current_player", np.int8, (B,)), ("move_count", np.int32, (B,)),
                         ("terminated", np.bool_, (B,)), ("truncated", np.bool_, (B,)),
                         ("outcome", np.int8, (B,)), ("seeds", np.uint64, (B,))):
        a = np.frombuffer(got[f], dt).reshape(shape)
        assert np.array_equal(a, want[f]), f
    stats = np.frombuffer(got["stats"], np.uint64)
    assert int(stats[0]) == steps and int(stats[5]) == B
    # lx_playout_host (host buffers only) plays the same episode
    assert np.array_equal(np.frombuffer(got["host_outcome"], np.int8), want["outcome"])
    assert np.array_equal(np.frombuffer(got["host_move_count"], np.int32), want["move_count"])
    assert np.array_equal(np.frombuffer(got["host_stats"], np.uint64)[:6], stats[:6])

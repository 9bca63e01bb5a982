"""bench.py helpers that read committed ncu captures (CPU only): a capture of
another build of the game must not be reported as this build's traffic."""
import json

import bench


class _FakeGame:
    def __init__(self, name, key):
        self.info = {"name": name}
        self._key = key

    def lowered_key(self):
        return self._key


def _write_step(tmp_path, key):
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "step_Fake_Game.json").write_text(json.dumps({
        "game": "fake", "batch": 1024, "cubin_key": key,
        "kernels": {"lx_random_step": {"dram_bytes_per_env": 96.5}}}))


def test_step_traffic_scales_to_batch(tmp_path, monkeypatch):
    _write_step(tmp_path, "abc")
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.step_traffic(_FakeGame("Fake Game", "abc"), "lx_random_step", 4096) == 96.5 * 4096


def test_step_traffic_stale_or_missing(tmp_path, monkeypatch):
    _write_step(tmp_path, "abc")
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.step_traffic(_FakeGame("Fake Game", "other"), "lx_random_step", 4096) is None
    assert bench.step_traffic(_FakeGame("Fake Game", "abc"), "lx_env_step", 4096) is None
    assert bench.step_traffic(_FakeGame("No Game", "abc"), "lx_random_step", 4096) is None


def test_rollout_profile_marks_stale(tmp_path, monkeypatch):
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "rollout_Fake_Game.json").write_text(json.dumps({"cubin_key": "abc",
                                                              "alu_warp_inst_per_env_step": 5.0}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.load_profile(_FakeGame("Fake Game", "abc"))["stale"] is False
    assert bench.load_profile(_FakeGame("Fake Game", "xyz"))["stale"] is True
    assert bench.load_profile(_FakeGame("No Game", "abc")) is None


def test_e2e_roofline_takes_the_slower_of_rollout_and_upload(monkeypatch):
    """e2e roofline = min(device rollout, seed upload at the PCIe peak): C4 is
    rollout-bound, TTT at 2^22 upload-bound (8 B per env per episode)."""
    monkeypatch.setattr(bench, "_PCIE_GBS", 50.0)
    B = 1 << 22
    c4 = {"value": 100e9, "h2d_bytes_per_step": 8 * B}
    rl = bench.e2e_roofline(c4, 21.3 * B, 110e9)          # 0.376 B/env step -> 133 G bound
    assert rl["bound"] == "device_rollout" and abs(rl["peak"] - 110e9) < 1
    assert abs(rl["frac"] - 100 / 110) < 1e-9
    assert abs(rl["pcie_h2d"]["bound_env_steps_per_s"] - 50e9 / (8 / 21.3)) < 1e3
    ttt = {"value": 40e9, "h2d_bytes_per_step": 8 * B}
    rl = bench.e2e_roofline(ttt, 7.6 * B, 134e9)           # 1.05 B/env step -> 47.5 G bound
    assert rl["bound"] == "pcie_h2d" and abs(rl["peak"] - 50e9 * 7.6 / 8) < 1e3
    assert bench.e2e_roofline("headline e2e", 1.0, 1.0) is None


def test_bench_table_reads_the_committed_bench_line(capsys):
    import runpy
    import sys
    argv = sys.argv
    import os
    sys.argv = ["bench_table.py", os.path.join(bench.ROOT, "profiles", "r2cert_bench.json")]
    try:
        runpy.run_path(os.path.join(bench.ROOT, "tools", "bench_table.py"), run_name="__main__")
    finally:
        sys.argv = argv
    out = capsys.readouterr().out
    assert "configs[1] C4" in out and "headline" in out

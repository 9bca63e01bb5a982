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

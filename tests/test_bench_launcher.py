"""bench.py's multi-process plumbing on CPU (gloo, world size 2): the self-
launch under torch.distributed.run when --gpus N > 1 arrives without
torchrun, one JSON line from rank 0 only, max-over-ranks timing, and the
workload description both arms print (identical by construction)."""
import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_launch_ranks_two_gloo_ranks_one_line():
    worker = os.path.join(HERE, "helpers", "launcher_worker.py")
    code = f"import sys; sys.path.insert(0, {ROOT!r}); import bench; sys.exit(bench.launch_ranks(2, {worker!r}, []))"
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")})
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["world"] == 2 and rec["ok"] and rec["total"] == rec["want_total"]
    assert rec["max_elapsed_ge"]  # the slowest rank's time is the one reported


def test_gpus_without_torchrun_relaunches(monkeypatch):
    seen = {}

    def fake(nproc, script, argv, env_extra=None):
        seen.update(nproc=nproc, script=script, argv=list(argv))
        return 0

    monkeypatch.setattr(bench, "launch_ranks", fake)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.main(["--gpus", "4", "--scaling", "strong", "--steps", "3"]) == 0
    assert seen["nproc"] == 4 and seen["script"].endswith("bench.py")
    assert seen["argv"] == ["--gpus", "4", "--scaling", "strong", "--steps", "3"]


def test_reference_arm_other_ranks_exit_quietly(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--impl", "reference", "--gpus", "2"]) == 0
    assert capsys.readouterr().out == ""


@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
@pytest.mark.parametrize("gpus,scaling", [(1, "weak"), (2, "weak"), (8, "weak"), (4, "strong"), (8, "strong")])
def test_config_dict_is_workload_only(name, gpus, scaling):
    cfg = bench.CONFIGS[name]
    d = bench.bench_config(cfg, gpus, scaling)
    assert d == bench.bench_config(dict(cfg), gpus, scaling)
    assert d["workload"] == cfg["desc"] and d["gpus"] == gpus and d["scaling"] == scaling
    if scaling == "weak":
        assert d["elements"] == cfg["n"] * gpus and d["elements_per_gpu"] == cfg["n"]
    else:
        assert d["elements"] == cfg["n"] and d["elements_per_gpu"] * gpus >= cfg["n"]


def test_launch_count_model():
    assert bench.launches_sharded(True, False, 0) == 2
    assert bench.launches_sharded(True, True, 3) == 3
    assert bench.launches_sharded(False, False, 0) == 1
    assert bench.launches_sharded(False, False, 2) == 2
    assert bench.launches_sharded(False, True, 2) == 4


def test_known_total_is_the_survey_value():
    # the reference engine's total on the exact cfg5 input
    assert bench.KNOWN_TOTALS["cfg5"] == 1073746006907

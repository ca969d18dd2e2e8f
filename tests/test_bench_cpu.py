"""bench.py's reference arm on the CPU (the driver runs `bench.py --impl
reference` beside our arm and computes the ratio from the two lines): one
JSON line with the same metric, unit and workload string as our arm, the
reference's own CPU implementation (oracle/_ref, run_moe_ll) timed on a
bounded token sample, steps and warm-up honoured; under torchrun only rank 0
prints.  Tiny sizes so the CPU suite stays fast."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _check_reference_line(d, ranks, tokens, steps, warmup):
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["higher_is_better"] is True
    assert d["config"]["workload"] == bench.workload(ranks, tokens)  # the string our arm prints
    assert d["config"]["ranks"] == ranks and d["config"]["sample_tokens_per_rank"] <= tokens
    assert d["steps"] == steps and d["warmup"] == warmup and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": bench.UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (reference sources absent)")
def test_reference_arm_line_single_process():
    env = dict(os.environ, GINSIM_REF_BUDGET_S="30")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--tokens", "64",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout
    _check_reference_line(lines[0], 8, 64, 2, 1)  # N=1: the 8-rank config, as our arm emulates it


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (reference sources absent)")
def test_reference_arm_under_torchrun_prints_once():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, GINSIM_REF_BUDGET_S="30")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--tokens", "64", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout  # rank 0 alone runs and prints; the other rank exits 0
    _check_reference_line(lines[0], 2, 64, 1, 1)
    assert lines[0]["n_gpus"] == 2


def test_step_bytes_and_workload_strings():
    """The metric's byte count: every (token, k) message of every rank, dispatch (2H+16) plus combine (2H)."""
    assert bench.step_bytes(8, 4096) == 8 * 4096 * 8 * ((2 * 7168 + 16) + 2 * 7168)
    assert bench.workload(8, 4096) == ("DeepEP HT dispatch+combine: 8 ranks x 4096 tokens/rank, hidden 7168, "
                                       "top-8 of 256 experts, u16 reference arithmetic")


def test_launch_count_claim_follows_the_library_plan(monkeypatch):
    import types
    a = types.SimpleNamespace(engine=0)
    assert bench.launches_per_step(a, 1, 8, 4096, 8, 256) == 3   # N=1: emulated ranks, no early reducer
    assert bench.launches_per_step(a, 4, 1, 4096, 8, 256) == 4   # NVLink: + the early reducer
    assert bench.launches_per_step(a, 4, 1, 128, 8, 256) == 3    # LL-sized: local route tables
    monkeypatch.setenv("GINSIM_COMBINE_CHUNKS", "0")
    assert bench.launches_per_step(a, 4, 1, 4096, 8, 256) == 3
    assert bench.launches_per_step(types.SimpleNamespace(engine=1), 4, 1, 4096, 8, 256) == 2

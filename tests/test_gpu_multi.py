"""Multi-GPU parity (world size 2 / 4 over NCCL): the P-rank step equals the
centralized step of the union batch (the reference's worker-count invariance)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world, placement):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, SPD_PLACEMENT=placement)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                          "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tests/multi_worker_impl.py")],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and lines, out.stdout[-3000:] + out.stderr[-3000:]
    return json.loads(lines[-1])


@pytest.mark.parametrize("placement", ["lbp", "seq", "local", "lbp-nct"])
def test_two_rank_step_matches_centralized(placement):
    r = _run(2, placement)
    if placement == "lbp-nct":  # replicated (NCT) and owned (CT) inverses in one step
        assert r["nct"] and len(r["nct"]) < 8, r
    assert r["identical_on_all_ranks"]
    assert max(r["errors"]) <= 1e-4, r
    assert r["bucketed"] and r["bucket_err"] <= 1e-5, r  # gradient bucket during backward == one all-reduce


def test_four_rank_step_matches_centralized():
    r = _run(4, "lbp")
    assert r["identical_on_all_ranks"]
    assert max(r["errors"]) <= 1e-4, r
    assert r["bucketed"] and r["bucket_err"] <= 1e-5, r

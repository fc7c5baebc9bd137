"""Multi-process (world size 2, gloo, CPU) coverage of the data-parallel host
logic, plus properties of the DDP bucket plan (-m "not gpu")."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def be():
    import paper_1912_01703_b200 as be
    from paper_1912_01703_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1912_01703_b200 import build
        build.build()
    return be


def test_ddp_plan_properties(be):
    numels = [int(np.prod(s[1])) for s in be.nn.ResNet50().param_specs()]
    bb = 25 << 20
    bof, off, bnum = be.ddp_plan(numels, bb)
    n = len(numels)
    assert len(bof) == n and all(b >= 0 for b in bof)
    # reverse registration order: bucket index is non-increasing with param index
    assert all(bof[i] >= bof[i + 1] for i in range(n - 1))
    assert bof[-1] == 0
    for b in range(len(bnum)):
        members = sorted((off[i], numels[i]) for i in range(n) if bof[i] == b)
        for (o1, n1), (o2, _) in zip(members, members[1:]):
            assert o1 + n1 <= o2  # no overlap
        assert all(o % 64 == 0 for o, _ in members)  # 256-B aligned views
        assert members[-1][0] + members[-1][1] == bnum[b]
        if b < len(bnum) - 1:
            assert bnum[b] * 4 >= bb  # every bucket but the last is full
    assert sum(numels) == 25557032
    assert len(bnum) == -(-sum(numels) * 4 // bb) or len(bnum) == sum(numels) * 4 // bb + 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_data_parallel_logic(tmp_path, be):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), str(tmp_path)]
    env = dict(os.environ, OMP_NUM_THREADS="1", PYTHONPATH=ROOT)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    res = [json.load(open(tmp_path / f"rank{i}.json")) for i in range(2)]
    for x in res:
        assert x["world"] == 2 and x["ok_uid"] and x["same_plan"] and x["replicas_equal"]
        assert x["err_emu"] < 1e-12 and x["err_glob"] < 1e-12
        assert x["tmax"] == 11.0

"""The library's own NCCL strip path (capi.cu: xfill / xfold / xallreduce captured in the CUDA
graph, nccl_shim.cu) executed by real processes, one per rank, all on the one GPU of the test box:
liblfsr loads the NCCL test double tests/fake_nccl (LFSR_NCCL_LIB), which implements Send / Recv /
AllReduce / Broadcast with CUDA IPC.  Every rank must return the same x as the single-strip solve
(<= 1e-5 relative L2, SURVEY §8c.4 multi-GPU bar) and the fp64 oracle (<= 1e-4 per iterate); the
timings are not measurements (the ranks time-share one GPU)."""
import json
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import lfsr_synth as S
from test_gpu_parity import oparams, rel_l2, ITER_TOL

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _tile_kernel_reference(monkeypatch):
    """The single-strip reference runs the same operator implementation as the strips (the fused
    tile kernel), so the comparison isolates the decomposition (the assembled operator, which only
    a single strip uses, is compared with the tile kernel in test_gpu_asm.py)."""
    monkeypatch.setenv("LFSR_ASM", "0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RANK_SCRIPT = textwrap.dedent(r'''
    import json, os, sys
    import numpy as np
    sys.path.insert(0, os.environ["LFSR_ROOT"])
    import lfsr_synth as S
    import paper_2206_05047_b200 as L
    cfg, n_ranks, rank, n_iters, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    uid = bytes.fromhex(os.environ["LFSR_TEST_UID"])
    lf = S.make_lightfield(cfg)
    p = L.params_for(S.CONFIGS[cfg], S.defaults_for(cfg), n_ranks=n_ranks, rank=rank, nccl_unique_id=uid)
    s = L.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    xs, stats = [s.get_hr()], []
    for _ in range(n_iters):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    st = s.get_state()
    s.close()
    np.savez(out, xs=np.array(xs), wA=st["wA"], wS=st["wS"])
    json.dump(stats, open(out + ".json", "w"))
''')


def run_ranks(cfg, n_ranks, n_iters, tmp_path):
    from tests_fake_nccl import lib_path
    env = dict(os.environ, LFSR_ROOT=ROOT, LFSR_NCCL_LIB=lib_path(), LFSR_TEST_UID=os.urandom(128).hex(),
               PYTHONPATH=ROOT)
    script = tmp_path / "rank.py"
    script.write_text(RANK_SCRIPT)
    procs = []
    for r in range(n_ranks):
        out = str(tmp_path / ("rank%d" % r))
        procs.append((subprocess.Popen([sys.executable, str(script), cfg, str(n_ranks), str(r), str(n_iters), out],
                                       env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), out))
    res = []
    for pr, out in procs:
        try:
            log = pr.communicate(timeout=600)[0].decode(errors="replace")
        except subprocess.TimeoutExpired:
            for q, _ in procs:
                q.kill()
            pytest.fail("NCCL-path ranks timed out")
        assert pr.returncode == 0, log[-3000:]
        z = np.load(out + ".npz")
        res.append((z["xs"], z["wA"], z["wS"], json.load(open(out + ".json"))))
    return res


def single_strip(L, cfg, n_iters):
    lf = S.make_lightfield(cfg)
    p = L.params_for(S.CONFIGS[cfg], S.defaults_for(cfg))
    s = L.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    xs, stats = [s.get_hr()], []
    for _ in range(n_iters):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    st = s.get_state()
    s.close()
    return p, lf, np.array(xs), stats, st


@pytest.mark.parametrize("cfg,n_ranks,n_iters", [("C1", 2, 4), ("C2", 2, 2), ("C2", 3, 2)])
def test_nccl_path_processes_match_single_strip(lfsr_mod, tmp_path, cfg, n_ranks, n_iters):
    import oracle as O
    p, lf, xs1, st1, s1 = single_strip(lfsr_mod, cfg, n_iters)
    res = run_ranks(cfg, n_ranks, n_iters, tmp_path)
    ora = O.admm(oparams(p), lf.y, lf.view_offsets, lf.omega, n_iters) if cfg == "C1" else None
    for r, (xs, wA, wS, stats) in enumerate(res):
        errs = [rel_l2(xs[i], xs1[i]) for i in range(n_iters + 1)]
        print("PARITY nccl-fake %s ranks=%d rank %d vs single strip: %s" % (
            cfg, n_ranks, r, " ".join("%.1e" % e for e in errs)))
        assert max(errs) <= 1e-5, errs
        for a, b in zip(stats, st1):
            assert a["cg_iters"] == b["cg_iters"]
            assert abs(a["J"] - b["J"]) <= 1e-6 * abs(b["J"])
        assert rel_l2(wA, s1["wA"]) <= 1e-5 and rel_l2(wS, s1["wS"]) <= 1e-4
        if ora is not None:
            eo = [rel_l2(xs[i], ora.x_iters[i]) for i in range(n_iters + 1)]
            assert max(eo) <= ITER_TOL, eo

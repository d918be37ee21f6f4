"""l(theta) on the paper's 2-D jittered grid at n = 20k / 40k against committed ORACLE
goldens (tests/golden/loglik_n*.json + z_n*.npy, written by tools/make_golden_large.py,
which calls only oracle/), through the production large-n launch path: CUDA graphs off,
the lookahead schedule, nb = 512, 1024 and 2048 (the bench's tile size at 100k).

Workload: Alg. 2 on the jittered grid of P:842-847, z = L(theta_true) e by the
oracle's Alg. 1; theta = the paper's Monte-Carlo theta (1, 0.1, 0.5) and a general-nu theta
(1, 0.1, 0.8) that runs the per-theta Chebyshev table of the generator.
Gates: plain |dl|/|l| <= 1e-10 and R13 (tests/_tol.py); logdet and quad <= 1e-10 relative.
"""
import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1708_02835_b200 as ex  # noqa: E402
from tests._tol import assert_ll  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(glob.glob(os.path.join(GOLDEN, "loglik_n*.json")))


def load(path):
    g = json.load(open(path))
    z = np.load(os.path.join(GOLDEN, f"z_n{g['n']}.npy"))
    assert z.shape == (g["n"],)
    return g, z


def test_goldens_present():
    ns = {json.load(open(f))["n"] for f in FILES}
    assert {20000, 40000} <= ns, ns


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
@pytest.mark.parametrize("nb", [512, 1024, 2048])
def test_loglik_matches_large_golden(path, nb):
    g, z = load(path)
    n = g["n"]
    x, y = ex.gen_locations(n, g["seed"])
    with ex.Context(device=0, nb=nb, graphs=-1) as c:
        for case in g["cases"]:
            th = tuple(case["theta"])
            r = c.loglik(x, y, z, th)
            assert r.info["nb"] == nb
            ref = (case["loglik"], case["logdet"], case["quad"])
            rel = assert_ll(r.loglik, ref, n, what=(n, nb, th))
            assert r.logdet == pytest.approx(case["logdet"], rel=1e-10)
            assert r.quad == pytest.approx(case["quad"], rel=1e-10)
            print(f"n={n} nb={nb} theta={th}: |dl|/|l| = {rel:.2e} (oracle {case['oracle_seconds']:.0f} s "
                  f"on {g['oracle_threads']} threads, GPU {r.info['ms_total']:.1f} ms)")

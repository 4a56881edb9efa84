"""The A/B switches.  MPID_FUSED_REFLECT runs the pass reduction and the reflector as one
launch (k_reduce_reflect); the fallback switches (MPID_ERR_NO_WS, MPID_NN_NO_WS, MPID_TN_NO_PIPE8) force the fp64
kernels the library takes for odd / unaligned shapes (register-staged error, NN-store Q1,
16-row TN tiles) on an aligned problem.  They are read once per process, so each
runs in a subprocess; every one must give the LSQ coefficients to 1e-10 and the
fused error (Remark 2) to 1e-9 against the oracle on the same skeleton.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.id import coeffs_lsq, id_error

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from tests.gpu_helpers import run_gpu
rng = np.random.default_rng(11)
m, n, k = 6144, 300, 100
A = np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 20.0)[None, :])
out = run_gpu(A, "fp32", "none", k, nb=4)
print(json.dumps({"piv": [int(i) for i in out["piv"]], "P": out["P"].tolist(), "err": list(out["err"])}))
"""


def _matrix():
    rng = np.random.default_rng(11)
    m, n = 6144, 300
    return np.asfortranarray(rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 20.0)[None, :])


@pytest.mark.parametrize("switch", [None, "MPID_ERR_NO_WS", "MPID_NN_NO_WS", "MPID_TN_NO_PIPE8", "MPID_FUSED_REFLECT"])
def test_switch_matches_oracle(switch):
    env = dict(os.environ)
    for s in ("MPID_ERR_NO_WS", "MPID_NN_NO_WS", "MPID_TN_NO_PIPE8", "MPID_FUSED_REFLECT"):
        env.pop(s, None)
    if switch:
        env[switch] = "1"
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    A = _matrix()
    I = np.asarray(got["piv"])
    P = np.asarray(got["P"])
    P_ref = coeffs_lsq(A, I)
    assert np.linalg.norm(P - P_ref) <= 1e-10 * np.linalg.norm(P_ref)
    e = id_error(A, I, P)
    assert abs(got["err"][0] - e[0]) <= 1e-9 * e[0]
    if switch == "MPID_FUSED_REFLECT":   # the same arithmetic per column: the same skeleton as the default
        r0 = subprocess.run([sys.executable, "-c", CHILD, ROOT], env={k: v for k, v in env.items() if k != switch},
                            capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r0.returncode == 0, r0.stderr[-2000:]
        assert json.loads(r0.stdout.strip().splitlines()[-1])["piv"] == got["piv"]

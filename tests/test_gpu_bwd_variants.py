"""The experimental backward variants (S2_DKV_V2: dK/dV over 128-row q steps;
S2_DQ_V2: dQ over 128-key steps; S2_PREP_FUSED: the prep fused into a dQ kernel
that runs before dK/dV), off by default because they are slower
at cfg3, against the oracle on the backward parity cases,
so the code that stays in the library is checked like the default path."""
import os

import numpy as np
import pytest

from test_gpu_bwd import CASES, TOL, run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env", ["S2_DKV_V2", "S2_DQ_V2", "S2_PREP_FUSED"])
@pytest.mark.parametrize("name", list(CASES))
def test_variant_matches_oracle(env, name):
    cfg, batch, D = CASES[name]
    os.environ[env] = "1"
    try:
        got, ref, _ = run(cfg, batch, D, seed=3)
    finally:
        del os.environ[env]
    for nm, g, r in zip(("dq", "dk", "dv"), got, ref):
        np.testing.assert_allclose(g, r, **TOL, err_msg=f"{env} {nm}")

"""K10 EvictionNet training against the reference trainer (net.py:107-279):
histories, early-stopping epochs and final parameters on reference-made
fixtures (tests/golden/make_trainnet_golden.py).  Float64 throughout; the
GEMM summation order and exp's last ulp differ from numpy, so the bar is a
tolerance: rtol 1e-9 on the MSE histories, rtol 1e-7 / atol 1e-10 on the
parameters, identical best / stopped epochs."""
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

import paper_2601_17063_b200 as mcb  # noqa: E402
from paper_2601_17063_b200 import train  # noqa: E402

Z = np.load(os.path.join(GOLDEN, "trainnet_cases.npz"))
META = json.loads(str(Z["meta"]))


def flat(net):
    return net.flat_params()


@pytest.mark.parametrize("case", META, ids=[m["name"] for m in META])
def test_training_matches_reference(case):
    k = case["name"]
    net = mcb.EvictionNet(case["E"], hidden=case["hidden"], seed=case["net_seed"])
    res = train.train_eviction_net(net, Z[k + "_f"], Z[k + "_t"], Z[k + "_m"], train.TrainConfig(**case["cfg"]))
    assert res.best_epoch == case["best_epoch"] and res.stopped_epoch == case["stopped_epoch"]
    np.testing.assert_allclose(res.train_mse, case["train_mse"], rtol=1e-9, atol=0)
    np.testing.assert_allclose(res.val_mse, case["val_mse"], rtol=1e-9, atol=0)
    np.testing.assert_allclose(flat(res.net), Z[k + "_params"], rtol=1e-7, atol=1e-10)


def test_batched_training_equals_one_at_a_time():
    cases = [m for m in META if m["name"].startswith("tn_e8_l")]
    cfg = train.TrainConfig(**cases[0]["cfg"])
    nets = [mcb.EvictionNet(c["E"], hidden=c["hidden"], seed=c["net_seed"]) for c in cases]
    data = [(Z[c["name"] + "_f"], Z[c["name"] + "_t"], Z[c["name"] + "_m"]) for c in cases]
    batched = train.train_eviction_nets(nets, data, cfg)
    for c, d, r in zip(cases, data, batched):
        single = train.train_eviction_net(mcb.EvictionNet(c["E"], hidden=c["hidden"], seed=c["net_seed"]), *d, cfg)
        assert r.train_mse == single.train_mse and r.val_mse == single.val_mse   # deterministic, no float atomics
        assert np.array_equal(flat(r.net), flat(single.net))


def test_non_finite_loss_raises_like_reference():
    c = META[0]
    f = np.array(Z[c["name"] + "_f"])
    f[5, 0] = np.nan
    net = mcb.EvictionNet(c["E"], hidden=c["hidden"], seed=0)
    with pytest.raises(train.NonFiniteLossError, match=r"non-finite loss nan at epoch 1, batch offset \d+"):
        train.train_eviction_net(net, f, Z[c["name"] + "_t"], Z[c["name"] + "_m"], train.TrainConfig(epochs=2))

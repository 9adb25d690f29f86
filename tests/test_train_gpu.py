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


def test_efficacy_net_retrained_on_gpu():
    """End to end (test_acceptance.py:223-275): the efficacy net is retrained on
    the GPU from GPU-generated traces and GPU training data, and compared with
    the reference-trained checkpoint (tests/golden/efficacy_net.evnet) and its
    held-out hit rates (ml 82.90 / lru 81.30 / lfu 79.78)."""
    from golden_util import load
    from paper_2601_17063_b200 import dataset, refgen
    from paper_2601_17063_b200.trace import TraceHeader
    header = TraceHeader("efficacy", 1, 64, 8)
    feats, targs, masks = [], [], []
    for s in (101, 102, 103):
        cfg = refgen.SyntheticWorkloadConfig(num_seqs=8, decode_steps=2500, prefill_tokens=32, zipf_s=1.0,
                                             recency_boost=0.3, w_hot=4, rng_seed=s, popularity_seed=7)
        ds = dataset.build_training_data(refgen.generate_trace(header, cfg), 64, 64)[0]
        feats.append(ds.features)
        targs.append(ds.targets)
        masks.append(ds.masks)
    net = mcb.EvictionNet(64, seed=0)
    res = train.train_eviction_net(net, np.concatenate(feats), np.concatenate(targs), np.concatenate(masks),
                                   train.TrainConfig(seed=0))
    ref = mcb.load_net(os.path.join(GOLDEN, "efficacy_net.evnet"))
    np.testing.assert_allclose(flat(res.net), ref.flat_params(), rtol=1e-6, atol=1e-9)
    import oracle
    from golden_util import case_trace
    rates = []
    for case in load("efficacy_cases.json.gz")["cases"]:
        header_, events = case_trace(case)
        from paper_2601_17063_b200.trace import AccessEvent, Phase, RoutingTrace
        L, E, K = header_
        tr = RoutingTrace(TraceHeader("e", L, E, K),
                          tuple(AccessEvent(s, Phase(p), t, l, tuple(x)) for s, p, t, l, x in events))
        rates.append(mcb.simulate(tr, "ml", 32, nets=res.net).hit_rate)
    assert round(100 * float(np.mean(rates)), 2) == 82.90

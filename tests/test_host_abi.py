"""CPU-side checks of the product library (no GPU needed).

* libpbkd_b200.so loads and exports every symbol include/pbkd_b200.h declares;
* the host-side, bit-exact parts of the hot path (seed derivation, split,
  epoch shuffles = activation indexing, candidate init, WFD/RR/makespan,
  MAC-proxy weights) equal the oracle bit for bit.
"""
import os
import re

import numpy as np
import pytest

import paper_2012_03096_b200 as P
from tests.conftest import ROOT, spec_text


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(P.LIB_PATH):
        P.build()


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "pbkd_b200.h")).read()
    declared = set(re.findall(r"\b(pbkd_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) > 30
    L = P.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name


def test_mix_seed_and_shuffle_match_oracle(orc):
    for a, b in [(42, 0), (42, 7), (2**63 + 5, 123456789)]:
        assert P.mix_seed(a, b) == orc.mix_seed(a, b)
    lab = (np.arange(1000) % 10).astype(np.int32)
    tr, ev = P.stratified_split(lab, 0.1, P.mix_seed(42, 0x5711))
    tr2, ev2 = orc.stratified_split(lab, 0.1, orc.mix_seed(42, 0x5711))
    assert np.array_equal(tr, tr2) and np.array_equal(ev, ev2)
    for epoch in (1, 2, 30):
        seed = P.mix_seed(42, 3)
        want = orc.shuffle(tr, orc.mix_seed(seed, epoch))  # distill.cpp:198-200
        assert np.array_equal(P.epoch_order(tr, seed, epoch), want)


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_candidate_init_bit_exact(orc, kind):
    # (256, 512, 2) / (512, 512, 1): tensors above he_fill's two-pass threshold
    for (cin, cout, s) in [(3, 64, 1), (64, 128, 2), (16, 16, 1), (256, 512, 2), (512, 512, 1)]:
        assert np.array_equal(P.build_candidate(kind, cin, cout, s, 99),
                              orc.build_candidate(kind, cin, cout, s, 99))


def test_scheduler_bit_exact(orc):
    rng = np.random.default_rng(0)
    for _ in range(50):
        n, w = int(rng.integers(1, 18)), int(rng.integers(1, 9))
        ids = list(range(1, n + 1))
        wt = rng.uniform(0.5, 20.0, n)
        plan, mk = P.wfd_bin_pack(ids, wt, w)
        plan2, mk2 = orc.wfd(ids, wt, w)
        assert plan == plan2 and mk == mk2
        assert P.round_robin(ids, w) == orc.round_robin(ids, w)
    # worked example (test_scheduler.cpp:30-60)
    ids, wt = [1, 2, 3, 4, 5], [8.0, 7.0, 6.0, 5.0, 4.0]
    assert P.makespan(P.round_robin(ids, 2), ids, wt) == 18.0
    assert P.makespan(P.wfd_bin_pack(ids, wt, 2)[0], ids, wt) == 17.0
    with pytest.raises(ValueError):
        P.wfd_bin_pack([1, 1], [1.0, 2.0], 1)
    with pytest.raises(ValueError):
        P.round_robin([1], 0)


def test_mac_proxy_weights_match_cost_model(orc):
    for name in ("vgg16_cifar", "resnet18_cifar", "toy_teacher"):
        spec = spec_text(name)
        nb = P.spec_num_blocks(spec)
        w = P.mac_proxy_weights(spec, list(range(1, nb + 1)))
        for k in range(1, nb + 1):
            assert w[k - 1] == orc.block_macs(spec, k) * 1e-6


def test_spec_errors_map_to_exceptions():
    with pytest.raises(ValueError):
        P.spec_num_blocks('{"input_shape": [3, 8, 8], "blocks": []}')
    with pytest.raises(ValueError):
        P.spec_num_blocks('{"input_shape": [3, 8, 8], "blocks": [{"kind": "conv5x5", '
                          '"out_channels": 4}], "classifier": [{"kind": "dense", "out_features": 2}]}')
    assert P.spec_num_floats(spec_text("toy_teacher")) == 14906

"""CPU tests of the seeded input generator (slcgen) — no GPU needed."""
import numpy as np
import pytest

import slcgen
from slcgen import gen


def test_deterministic_and_shard_independent():
    a = slcgen.generate(slcgen.WHAT_THETA_LOCAL, 7, 3, 1000, 5000, special_period=16)
    b = slcgen.generate(slcgen.WHAT_THETA_LOCAL, 7, 3, 1000, 5000, special_period=16)
    assert (a.view(np.uint32) == b.view(np.uint32)).all()
    # any sub-range reproduces the same values (keyed on the global index)
    c = slcgen.generate(slcgen.WHAT_THETA_LOCAL, 7, 3, 3000, 1000, special_period=16)
    assert (a[2000:3000].view(np.uint32) == c.view(np.uint32)).all()
    # peers differ, theta does not depend on the peer
    d = slcgen.generate(slcgen.WHAT_THETA_LOCAL, 7, 4, 1000, 5000)
    assert (a != d).any()
    t3 = slcgen.generate(slcgen.WHAT_THETA, 7, 3, 0, 8192, special_period=4)
    t4 = slcgen.generate(slcgen.WHAT_THETA, 7, 4, 0, 8192, special_period=4)
    assert (t3.view(np.uint32) == t4.view(np.uint32)).all()


def test_value_ranges():
    n = 1 << 16
    th = slcgen.generate(slcgen.WHAT_THETA, 0, 0, 0, n)
    tl = slcgen.generate(slcgen.WHAT_THETA_LOCAL, 0, 0, 0, n)
    ef = slcgen.generate(slcgen.WHAT_EF, 0, 0, 0, n, warm_ef=True)
    assert abs(th.std() - 0.02) < 0.001 and np.abs(th).max() <= 2 * 0.0347
    d = th.astype(np.float64) - tl
    assert np.abs(d).max() <= 2.0 ** -10 * 1.001 and (d != 0).mean() > 0.99
    assert np.abs(ef).max() <= 2.0 ** -8
    assert (slcgen.generate(slcgen.WHAT_EF, 0, 0, 0, n) == 0).all()


def test_special_families_present():
    n = 4096 * 512
    fam = gen.special_family(0, np.arange(0, n, 4096, dtype=np.uint64), 8)
    present = set(fam[fam >= 0].tolist())
    assert present == set(range(slcgen.N_FAMILIES))
    tl = slcgen.generate(slcgen.WHAT_THETA_LOCAL, 0, 0, 0, n, special_period=8)
    th = slcgen.generate(slcgen.WHAT_THETA, 0, 0, 0, n, special_period=8)
    runs = np.arange(n) >> 12
    sub_runs = np.nonzero(fam == 4)[0]
    d = th[np.isin(runs, sub_runs)] - tl[np.isin(runs, sub_runs)]
    assert (np.abs(d) < 2.0 ** -126).all() and (d != 0).any()   # fp32 subnormals


def test_bf16_bits_match_torch():
    torch = pytest.importorskip("torch")
    x = slcgen.generate(slcgen.WHAT_THETA, 1, 0, 0, 50000)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = slcgen.generate(slcgen.WHAT_THETA, 1, 0, 0, 50000, dtype="bf16")
    assert (got == ref).all()

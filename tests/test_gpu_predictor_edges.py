"""Arithmetic edges of the device predictor (k_predict.cu), written like the
reference's hand-built-descriptor tests (test_predictor.py:70-126) and
checked against the oracle's restatement of analyzer.py:112-174
(`oracle.msched_port.predict_template`), which the golden predictions pin
to the reference:

* exact rational coefficients (1/3, 7/2): integral products predict, a
  non-integral product makes the rule return None (analyzer.py:125-127), so
  the prediction is incomplete and keeps only the other rules' pages;
* `max(size, 1)` for zero and negative extents (analyzer.py:166);
* strided rules with count < 1 are None (analyzer.py:171-172);
* `unpredictable` rules and `unpredictable_fraction` mark incompleteness.

Where the device cannot compute what the reference computes it must say
so with MSG_E_DOMAIN rather than return a different set:
* a coefficient whose numerator or denominator needs more than 64 bits;
* a strided rule expanding to more than 2^24 chunks;
* a prediction outside every allocation, ground-truth range and memcpy
  extent of the Simulator's dense page map.
"""

from fractions import Fraction

import pytest

from oracle import msched_port as port
from paper_2512_24637_b200 import _abi, engine, predictor
from paper_2512_24637_b200.analyzer import KernelDescriptor, LinearExpr, TemplateRule
from paper_2512_24637_b200.model import Allocation, Arg, ByteRange, Command, CommandKind, HwConfig, Task
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scheduler import Policy

pytestmark = pytest.mark.gpu
PAGE = 4096
BASE = 1 << 30


def kcmd(args, grid=(1, 1, 1), block=(1, 1, 1), name="k"):
    return Command(CommandKind.KERNEL, 1e-6, name, tuple(args), grid, block)


def fixed(n, ptr=0, off=0):
    return TemplateRule(ptr, "fixed", off, size=LinearExpr(Fraction(n)))


def linear(coeff, slots, ptr=0, off=0):
    return TemplateRule(ptr, "linear", off, size=LinearExpr(Fraction(coeff), tuple(slots)))


def strided(stride, chunk, count, ptr=0, off=0):
    return TemplateRule(ptr, "strided", off, stride=LinearExpr(*stride), chunk=LinearExpr(*chunk),
                        count=LinearExpr(*count))


def both(desc, cmd):
    got = predictor.predict({"k": desc}, cmd, PAGE)
    runs, complete = port.predict_template({"k": desc}, cmd, PAGE)
    assert [tuple(r) for r in got.pages.runs] == [tuple(r) for r in runs]
    assert got.complete == complete
    return got


def test_fraction_coefficient_integral_and_not():
    d = KernelDescriptor("k", [linear(Fraction(1, 3), ["a1"])])
    p = both(d, kcmd([Arg(BASE), Arg(3 * PAGE, 32)]))            # 1/3 * 3P = P bytes
    assert p.complete and list(p.pages) == [BASE // PAGE]
    p = both(d, kcmd([Arg(BASE), Arg(3 * PAGE + 1, 32)]))        # non-integral -> None
    assert not p.complete and len(p.pages) == 0
    # a second rule still contributes when the first is non-integral
    d2 = KernelDescriptor("k", [linear(Fraction(1, 3), ["a1"]), fixed(2 * PAGE, ptr=2)])
    p = both(d2, kcmd([Arg(BASE), Arg(7, 32), Arg(BASE + 64 * PAGE)]))
    assert not p.complete and list(p.pages) == [BASE // PAGE + 64, BASE // PAGE + 65]


def test_fraction_products_of_several_slots_and_launch_dims():
    d = KernelDescriptor("k", [linear(Fraction(7, 2), ["a1", "gx", "bx"])])
    for a1, gx, bx in ((2, 3, 128), (5, 7, 64), (3, 1, 1), (1, 1, 1)):
        both(d, kcmd([Arg(BASE), Arg(a1, 32)], grid=(gx, 1, 1), block=(bx, 1, 1)))


def test_zero_and_negative_sizes_touch_one_byte():
    for n in (0, -5 * PAGE):
        p = both(KernelDescriptor("k", [fixed(n)]), kcmd([Arg(BASE + 100)]))
        assert p.complete and list(p.pages) == [BASE // PAGE]


def test_strided_counts_below_one_are_unpredictable():
    for count in (0, -3):
        d = KernelDescriptor("k", [strided((Fraction(2 * PAGE),), (Fraction(PAGE),), (Fraction(count),))])
        p = both(d, kcmd([Arg(BASE)]))
        assert not p.complete and len(p.pages) == 0
    d = KernelDescriptor("k", [strided((Fraction(3 * PAGE),), (Fraction(PAGE, 2),), (Fraction(1), ("a1",)))])
    p = both(d, kcmd([Arg(BASE), Arg(4, 32)]))
    assert p.complete and list(p.pages) == [BASE // PAGE + 3 * j for j in range(4)]


def test_unpredictable_rule_and_fraction_mark_incomplete():
    d = KernelDescriptor("k", [TemplateRule(0, "unpredictable"), fixed(PAGE)])
    p = both(d, kcmd([Arg(BASE)]))
    assert not p.complete and list(p.pages) == [BASE // PAGE]
    d = KernelDescriptor("k", [fixed(PAGE)], unpredictable_fraction=0.25)   # test_predictor.py:108-126
    p = both(d, kcmd([Arg(BASE)]))
    assert not p.complete and list(p.pages) == [BASE // PAGE]


def test_pointer_index_past_the_arguments_is_none():
    p = both(KernelDescriptor("k", [fixed(PAGE, ptr=3)]), kcmd([Arg(BASE)]))
    assert not p.complete and len(p.pages) == 0


def _code(fn):
    with pytest.raises(_abi.MsgError) as ei:
        fn()
    return ei.value.code


def test_coefficient_beyond_64_bits_is_domain():
    for coeff in (Fraction(1 << 63), Fraction(1, 1 << 64), Fraction(-(1 << 64), 3)):
        d = KernelDescriptor("k", [linear(coeff, ["a1"])])
        assert _code(lambda: predictor.predict({"k": d}, kcmd([Arg(BASE), Arg(1, 32)]), PAGE)) == _abi.MSG_E_DOMAIN


def test_strided_count_beyond_2_24_is_domain():
    d = KernelDescriptor("k", [strided((Fraction(PAGE),), (Fraction(1),), (Fraction((1 << 24) + 1),))])
    assert _code(lambda: predictor.predict({"k": d}, kcmd([Arg(BASE)]), PAGE)) == _abi.MSG_E_DOMAIN
    d = KernelDescriptor("k", [strided((Fraction(PAGE),), (Fraction(1),), (Fraction(1 << 10),))])
    p = both(d, kcmd([Arg(BASE)]))
    assert len(p.pages) == 1 << 10


def test_prediction_outside_the_dense_map_is_domain():
    """A planted rule pointing 1 GiB past the task's only allocation: the
    reference would plan those pages; the device refuses the command table
    (its dense page map covers allocations, ground truth and memcpy
    extents) instead of silently dropping them."""
    base = 1 << 40
    alloc = Allocation("a", base, 16 * PAGE, "t")
    cmds = [Command(CommandKind.KERNEL, 1e-5, "k", (Arg(base, 64),), ground_truth_access=(ByteRange(base, PAGE),))
            for _ in range(3)]
    task = Task("t", [alloc], cmds)
    desc = {"t": {"k": KernelDescriptor("k", [fixed(PAGE, off=1 << 30)])}}
    hw = get_preset("rtx5080").with_capacity(64 * PAGE)
    assert isinstance(hw, HwConfig)
    with pytest.raises(_abi.MsgError) as ei:
        engine.Simulator([task], hw, Policy("rr", 1e-3), engine.Mode.proactive(), descriptors=desc)
    assert ei.value.code == _abi.MSG_E_DOMAIN
    # inside the allocation the same rule shape replays and matches the oracle
    desc_ok = {"t": {"k": KernelDescriptor("k", [fixed(PAGE, off=4 * PAGE)])}}
    sim = engine.Simulator([task], hw, Policy("rr", 1e-3), engine.Mode.proactive(), descriptors=desc_ok)
    try:
        m = sim.run()
    finally:
        sim.close()
    assert m.completed_tasks == 1

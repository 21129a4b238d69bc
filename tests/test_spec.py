"""Spec grammar parity (reference tests/test_driver.py:54-110, test_dset.py:41-70,
test_minbased.py:52-69) — pure host logic, no GPU."""
import pytest

from paper_2008_11839_b200 import (LT_VARIANTS, AlgorithmSpec, ConfigError, FindOp, FinishKind,
                                   SampleKind, SpliceOp, UnionConfig, UnionOp, all_valid_configs,
                                   enumerate_specs, format_spec, parse_spec, valid_combination)
from paper_2008_11839_b200.spec import ConnectRule, LTVariant, ShortcutRule, UpdateRule, is_root_based


def test_every_spec_round_trips():
    specs = enumerate_specs()
    assert len(specs) == 204
    texts = [format_spec(s) for s in specs]
    assert len(set(texts)) == 204
    for s, t in zip(specs, texts):
        assert parse_spec(t) == s


def test_census(golden):
    specs = enumerate_specs()
    assert sum(s.is_union_finish() for s in specs) == 128
    assert sum(s.is_root_based() for s in specs) == 132
    assert sum(s.incremental_capable() and s.sample is SampleKind.NONE for s in specs) == 39
    # the reference's own spec list (golden keys) is exactly ours
    ref = set(next(iter(golden.spec_stats.values())).keys())
    assert ref == {format_spec(s) for s in specs}


def test_ldd_specs():
    s = parse_spec("ldd+sv")
    assert s.sample is SampleKind.LDD and s.ldd_beta == 0.2
    s2 = parse_spec("ldd(0.35)+lt_prs")
    assert s2.ldd_beta == 0.35 and format_spec(s2) == "ldd(0.35)+lt_prs"
    assert parse_spec(format_spec(s2)) == s2
    assert len(enumerate_specs(samples=list(SampleKind))) == 255


@pytest.mark.parametrize("text", [
    "xout+async+halve", "kout", "none+lt", "none+lt_zzz", "none+sv+halve",
    "none+async+halve+splice", "none+async+twotry", "none+rem_cas+compress+splice",
    "none+async+halve+extra+extra", "ldd(x)+sv", "none+rem_cas+naive+none"])
def test_malformed(text):
    with pytest.raises(ConfigError):
        parse_spec(text)


def test_defaults():
    assert parse_spec("none+rem_cas+naive").cfg.splice is SpliceOp.SPLICE_ATOMIC
    s2 = parse_spec("kout+async")
    assert s2.cfg.find is FindOp.NAIVE and s2.kout_k == 2
    assert parse_spec("none+async+halve", seed=9).seed == 9


def test_construction_validation():
    with pytest.raises(ConfigError):
        AlgorithmSpec(SampleKind.NONE, FinishKind.ASYNC, UnionConfig(UnionOp.HOOKS, FindOp.NAIVE))
    with pytest.raises(ConfigError):
        AlgorithmSpec(SampleKind.NONE, FinishKind.LT)


def test_matrix():
    cfgs = all_valid_configs()
    assert len(cfgs) == 32
    by = {}
    for c in cfgs:
        by.setdefault(c.union, []).append(c)
    assert [len(by[u]) for u in UnionOp] == [4, 4, 4, 9, 9, 2]
    assert not valid_combination(UnionConfig(UnionOp.REM_CAS, FindOp.COMPRESS, SpliceOp.SPLICE_ATOMIC))
    assert valid_combination(UnionConfig(UnionOp.JTB, FindOp.TWO_TRY))


def test_lt_variants():
    assert len(LT_VARIANTS) == 16
    assert {n for n, v in LT_VARIANTS.items() if is_root_based(v)} == {"crsa", "prsa", "prs", "crfa", "prfa", "prf"}
    with pytest.raises(ValueError):
        LTVariant("cus", ConnectRule.CONNECT, UpdateRule.ALL, ShortcutRule.ONE, alter=False)

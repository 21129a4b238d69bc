"""The algorithm-selection grammar of the drop-in surface.

Mirrors connlab's spec language (reference driver.py:65-307, dset.py:29-87,
minbased.py:24-84, sampling.py:19-26): a run is ``sample+finish[+find[+splice]]``
such as ``kout+rem_cas+halve+splice`` or ``bfs+lt_prs``.  Names, defaults,
validation rules and error type (ConfigError, raised before any work) are the
reference's; the one addition is the ``ldd`` sampler (optionally written
``ldd(beta)``) that the GConn north star asks for and the reference lacks.
"""
from __future__ import annotations

import re
from dataclasses import dataclass
from enum import Enum
from typing import Optional

from .errors import ConfigError


class SampleKind(Enum):
    NONE = "none"
    KOUT = "kout"
    HB = "hb"
    BFS = "bfs"
    LDD = "ldd"


# samplers of the reference (driver.py:65-69); enumerate_specs() defaults to these
REFERENCE_SAMPLES = (SampleKind.NONE, SampleKind.KOUT, SampleKind.HB, SampleKind.BFS)


class FinishKind(Enum):
    ASYNC = "async"
    HOOKS = "hooks"
    EARLY = "early"
    REM_LOCK = "rem_lock"
    REM_CAS = "rem_cas"
    JTB = "jtb"
    SV = "sv"
    LT = "lt"
    STERGIOU = "stergiou"
    LP = "lp"


class UnionOp(Enum):
    ASYNC = "async"
    HOOKS = "hooks"
    EARLY = "early"
    REM_LOCK = "rem_lock"
    REM_CAS = "rem_cas"
    JTB = "jtb"


class FindOp(Enum):
    NAIVE = "naive"
    SPLIT = "split"
    HALVE = "halve"
    COMPRESS = "compress"
    TWO_TRY = "twotry"


class SpliceOp(Enum):
    NONE = "none"
    SPLIT_ONE = "split"
    HALVE_ONE = "halve"
    SPLICE_ATOMIC = "splice"


class KOutMode(Enum):
    FIRST_K = "first_k"
    FIRST_PLUS_RANDOM = "first_plus_random"


KOUT_DEFAULT_K = 2       # sampling.py:19
HB_DEFAULT_EDGES = 4     # sampling.py:20
BFS_DEFAULT_PROBES = 64  # sampling.py:21
LDD_DEFAULT_BETA = 0.2   # new sampler (no reference default)


@dataclass(frozen=True)
class UnionConfig:
    union: UnionOp
    find: FindOp = FindOp.NAIVE
    splice: SpliceOp = SpliceOp.NONE


# The supported matrix (dset.py:60-76): allowed finds / splices per union rule.
_MATRIX = {
    UnionOp.ASYNC: ((FindOp.NAIVE, FindOp.SPLIT, FindOp.HALVE, FindOp.COMPRESS), (SpliceOp.NONE,)),
    UnionOp.HOOKS: ((FindOp.NAIVE, FindOp.SPLIT, FindOp.HALVE, FindOp.COMPRESS), (SpliceOp.NONE,)),
    UnionOp.EARLY: ((FindOp.NAIVE, FindOp.SPLIT, FindOp.HALVE, FindOp.COMPRESS), (SpliceOp.NONE,)),
    UnionOp.REM_LOCK: ((FindOp.NAIVE, FindOp.SPLIT, FindOp.HALVE),
                       (SpliceOp.SPLIT_ONE, SpliceOp.HALVE_ONE, SpliceOp.SPLICE_ATOMIC)),
    UnionOp.REM_CAS: ((FindOp.NAIVE, FindOp.SPLIT, FindOp.HALVE),
                      (SpliceOp.SPLIT_ONE, SpliceOp.HALVE_ONE, SpliceOp.SPLICE_ATOMIC)),
    UnionOp.JTB: ((FindOp.NAIVE, FindOp.TWO_TRY), (SpliceOp.NONE,)),
}


def valid_combination(cfg: UnionConfig) -> bool:
    finds, splices = _MATRIX[cfg.union]
    return cfg.find in finds and cfg.splice in splices


def all_valid_configs() -> list[UnionConfig]:
    """The 32 (union, find, splice) combinations, in enum order."""
    return [UnionConfig(u, f, s) for u in UnionOp for f in FindOp for s in SpliceOp
            if valid_combination(UnionConfig(u, f, s))]


# ---------------------------------------------------------------- Liu-Tarjan

class ConnectRule(Enum):
    CONNECT = "connect"
    PARENT = "parent_connect"
    EXTENDED = "extended_connect"


class UpdateRule(Enum):
    ALL = "update"
    ROOTS = "root_update"


class ShortcutRule(Enum):
    ONE = "shortcut"
    FULL = "full_shortcut"


@dataclass(frozen=True)
class LTVariant:
    name: str
    connect: ConnectRule
    update: UpdateRule
    shortcut: ShortcutRule
    alter: bool

    def __post_init__(self):
        # minbased.py:48-52: endpoint-id messages need the alter rewrite
        if self.connect is ConnectRule.CONNECT and not self.alter:
            raise ValueError(f"{self.name}: Connect requires the alter phase")


def _variant_from_name(name: str) -> LTVariant:
    """Variant names spell their rules: c/p/e connect, u/r update,
    s/f shortcut, trailing a = alter (minbased.py:59-79)."""
    connect = {"c": ConnectRule.CONNECT, "p": ConnectRule.PARENT, "e": ConnectRule.EXTENDED}[name[0]]
    update = {"u": UpdateRule.ALL, "r": UpdateRule.ROOTS}[name[1]]
    shortcut = {"s": ShortcutRule.ONE, "f": ShortcutRule.FULL}[name[2]]
    return LTVariant(name, connect, update, shortcut, name.endswith("a"))


_LT_NAMES = ["cusa", "crsa", "pusa", "prsa", "pus", "prs", "eusa", "eus",
             "cufa", "crfa", "pufa", "prfa", "puf", "prf", "eufa", "euf"]
LT_VARIANTS: dict[str, LTVariant] = {nm: _variant_from_name(nm) for nm in _LT_NAMES}


def is_root_based(variant: LTVariant) -> bool:
    return variant.update is UpdateRule.ROOTS


# ------------------------------------------------------------- AlgorithmSpec

_UNION_OF = {
    FinishKind.ASYNC: UnionOp.ASYNC, FinishKind.HOOKS: UnionOp.HOOKS,
    FinishKind.EARLY: UnionOp.EARLY, FinishKind.REM_LOCK: UnionOp.REM_LOCK,
    FinishKind.REM_CAS: UnionOp.REM_CAS, FinishKind.JTB: UnionOp.JTB,
}

# samplers run Async+Halve when the finish is not union-find (driver.py:96)
SAMPLER_FALLBACK = UnionConfig(UnionOp.ASYNC, FindOp.HALVE)


def _cfg_text(cfg: UnionConfig) -> str:
    parts = [cfg.union.value, cfg.find.value]
    if cfg.splice is not SpliceOp.NONE:
        parts.append(cfg.splice.value)
    return "+".join(parts)


def _default_union_cfg(union: UnionOp) -> UnionConfig:
    splice = SpliceOp.SPLICE_ATOMIC if union in (UnionOp.REM_LOCK, UnionOp.REM_CAS) else SpliceOp.NONE
    return UnionConfig(union, FindOp.NAIVE, splice)


@dataclass(frozen=True)
class AlgorithmSpec:
    sample: SampleKind = SampleKind.NONE
    finish: FinishKind = FinishKind.ASYNC
    cfg: Optional[UnionConfig] = None
    lt_variant: Optional[LTVariant] = None
    kout_k: int = KOUT_DEFAULT_K
    kout_mode: KOutMode = KOutMode.FIRST_K
    hb_edges: int = HB_DEFAULT_EDGES
    bfs_probes: int = BFS_DEFAULT_PROBES
    seed: int = 1
    ldd_beta: float = LDD_DEFAULT_BETA

    def __post_init__(self):
        union = _UNION_OF.get(self.finish)
        if union is not None:
            if self.cfg is None:
                object.__setattr__(self, "cfg", _default_union_cfg(union))
            if self.cfg.union is not union:
                raise ConfigError(f"finish '{self.finish.value}' does not match union rule "
                                  f"'{self.cfg.union.value}'")
            if not valid_combination(self.cfg):
                raise ConfigError(f"unsupported combination {_cfg_text(self.cfg)}; valid: "
                                  + ", ".join(_cfg_text(c) for c in all_valid_configs()))
        elif self.cfg is not None:
            raise ConfigError(f"finish '{self.finish.value}' takes no find/splice rules")
        if (self.finish is FinishKind.LT) != (self.lt_variant is not None):
            if self.lt_variant is None:
                raise ConfigError("lt finish requires a variant: " + ", ".join(sorted(LT_VARIANTS)))
            raise ConfigError(f"finish '{self.finish.value}' takes no lt variant")
        if self.kout_k < 1:
            raise ConfigError(f"kout_k must be >= 1, got {self.kout_k}")
        if self.hb_edges < 0 or self.bfs_probes < 1:
            raise ConfigError("hb_edges must be >= 0 and bfs_probes >= 1")
        if not (self.ldd_beta > 0):
            raise ConfigError(f"ldd_beta must be > 0, got {self.ldd_beta}")

    def is_union_finish(self) -> bool:
        return self.finish in _UNION_OF

    def is_root_based(self) -> bool:
        """Only roots are ever redirected (driver.py:145-154): forests can be recorded."""
        if self.is_union_finish():
            return self.cfg.splice is not SpliceOp.SPLICE_ATOMIC
        if self.finish is FinishKind.SV:
            return True
        if self.finish is FinishKind.LT:
            return is_root_based(self.lt_variant)
        return False

    def incremental_capable(self) -> bool:
        """driver.py:156-165: union-find (any splice), SV, root-based LT."""
        if self.is_union_finish() or self.finish is FinishKind.SV:
            return True
        return self.finish is FinishKind.LT and is_root_based(self.lt_variant)

    def sampler_config(self) -> UnionConfig:
        return self.cfg if self.is_union_finish() else SAMPLER_FALLBACK


_LDD_RE = re.compile(r"^ldd(?:\(([0-9]*\.?[0-9]+(?:e-?[0-9]+)?)\))?$")


def _finish_token_list() -> list[str]:
    return [k.value for k in FinishKind if k is not FinishKind.LT] + [f"lt_{n}" for n in LT_VARIANTS]


def parse_spec(text: str, **overrides) -> AlgorithmSpec:
    """Parse ``sample+finish[+find[+splice]]`` (driver.py:197-276)."""
    tokens = text.strip().lower().split("+")
    if len(tokens) < 2:
        raise ConfigError(f"spec '{text}' needs at least sample+finish; samples: "
                          + ", ".join(k.value for k in SampleKind)
                          + "; finishes: " + ", ".join(_finish_token_list()))
    head, ftok, rest = tokens[0], tokens[1], tokens[2:]
    mldd = _LDD_RE.match(head)
    if mldd:
        sample = SampleKind.LDD
        if mldd.group(1) is not None and "ldd_beta" not in overrides:
            overrides["ldd_beta"] = float(mldd.group(1))
    else:
        try:
            sample = SampleKind(head)
        except ValueError:
            raise ConfigError(f"unknown sampling '{head}'; valid: "
                              + ", ".join(k.value for k in SampleKind)) from None

    variant = None
    if ftok.startswith("lt_"):
        variant = LT_VARIANTS.get(ftok[3:])
        if variant is None:
            raise ConfigError(f"unknown lt variant '{ftok[3:]}'; valid: " + ", ".join(sorted(LT_VARIANTS)))
        finish = FinishKind.LT
    else:
        try:
            finish = FinishKind(ftok)
        except ValueError:
            raise ConfigError(f"unknown finish '{ftok}'; valid: " + ", ".join(_finish_token_list())) from None
        if finish is FinishKind.LT:
            raise ConfigError("lt finish needs a variant suffix, e.g. "
                              + ", ".join(f"lt_{n}" for n in sorted(LT_VARIANTS)))

    cfg = None
    union = _UNION_OF.get(finish)
    if union is not None:
        base = _default_union_cfg(union)
        find, splice = base.find, base.splice
        if rest:
            try:
                find = FindOp(rest[0])
            except ValueError:
                raise ConfigError(f"unknown find rule '{rest[0]}'; valid: "
                                  + ", ".join(f.value for f in FindOp)) from None
            rest = rest[1:]
        if rest:
            if rest[0] == SpliceOp.NONE.value:
                raise ConfigError("unknown splice rule 'none'")
            try:
                splice = SpliceOp(rest[0])
            except ValueError:
                raise ConfigError(f"unknown splice rule '{rest[0]}'; valid: split, halve, splice") from None
            rest = rest[1:]
        cfg = UnionConfig(union, find, splice)
        if not valid_combination(cfg):
            raise ConfigError(f"unsupported combination '{text}'; valid union combinations: "
                              + ", ".join(_cfg_text(c) for c in all_valid_configs()))
    if rest:
        raise ConfigError(f"trailing tokens {rest} in spec '{text}': finish '{ftok}' takes "
                          + ("find[+splice] only" if cfg is not None else "no further rules"))
    return AlgorithmSpec(sample=sample, finish=finish, cfg=cfg, lt_variant=variant, **overrides)


def format_spec(spec: AlgorithmSpec) -> str:
    if spec.finish is FinishKind.LT:
        fin = f"lt_{spec.lt_variant.name}"
    elif spec.is_union_finish():
        fin = _cfg_text(spec.cfg)
    else:
        fin = spec.finish.value
    head = spec.sample.value
    if spec.sample is SampleKind.LDD and spec.ldd_beta != LDD_DEFAULT_BETA:
        head = f"ldd({spec.ldd_beta:g})"
    return f"{head}+{fin}"


def enumerate_specs(samples=None) -> list[AlgorithmSpec]:
    """Every supported spec (driver.py:289-307): samplers x (32 union
    combinations, SV, 16 LT variants, Stergiou, LP).  Defaults to the four
    reference samplers (204 specs); pass samples=list(SampleKind) for LDD too."""
    if samples is None:
        samples = list(REFERENCE_SAMPLES)
    union_kind = {u: k for k, u in _UNION_OF.items()}
    finishes = [(union_kind[c.union], c, None) for c in all_valid_configs()]
    finishes.append((FinishKind.SV, None, None))
    finishes += [(FinishKind.LT, None, LT_VARIANTS[nm]) for nm in LT_VARIANTS]
    finishes += [(FinishKind.STERGIOU, None, None), (FinishKind.LP, None, None)]
    return [AlgorithmSpec(sample=s, finish=k, cfg=c, lt_variant=v) for s in samples for (k, c, v) in finishes]

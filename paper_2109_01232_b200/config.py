"""Run configuration of the experiment harness (reference io.py:208-368).

``RunConfig`` / ``SolverKind`` / ``PrecondSpec`` / ``ConfigError`` and the
``key = value`` grammar (``parse_run_config``, ``format_run_config``,
``load_run_config``) keep the reference's names, defaults, validation rules
and error messages, so a reference config file drives this package's CLI
(``python -m paper_2109_01232_b200``) and the sweeps in ``bench`` unchanged.
Host-only: nothing here touches the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .gen import RhsKind, RhsSpec, StencilSpec, parse_rhs_spec, parse_stencil_spec

__all__ = ["ConfigError", "SolverKind", "PrecondSpec", "RunConfig", "FP32_RTOL_FLOOR",
           "parse_run_config", "format_run_config", "load_run_config"]

FP32_RTOL_FLOOR = 1e-6          # io.py:48: an fp32 solve cannot target tighter


class ConfigError(ValueError):
    """Invalid run configuration (io.py:55-56)."""


class SolverKind(Enum):
    """io.py:211-215."""
    DOUBLE = "double"
    SINGLE = "single"
    IR = "ir"
    FD = "fd"


@dataclass(frozen=True)
class PrecondSpec:
    """``none``, ``jacobi:K`` (block size) or ``poly:D`` (degree) (io.py:218-241)."""

    kind: str = "none"
    param: int = 0

    def __str__(self) -> str:
        return self.kind if self.kind == "none" else f"{self.kind}:{self.param}"

    @classmethod
    def parse(cls, text: str) -> "PrecondSpec":
        text = text.strip().lower()
        if text in ("", "none"):
            return cls()
        name, _, param = text.partition(":")
        if name not in ("jacobi", "poly") or not param:
            raise ConfigError(f"bad preconditioner {text!r}; expected none, jacobi:K, or poly:D")
        value = int(param)
        if name == "jacobi" and value < 1:
            raise ConfigError("block size must be positive")
        if name == "poly" and value < 0:
            raise ConfigError("polynomial degree must be nonnegative")
        return cls(name, value)


@dataclass
class RunConfig:
    """Full description of one experiment (io.py:244-281)."""

    solver: SolverKind
    matrix: str | None = None
    gen: StencilSpec | None = None
    m: int = 50
    rtol: float = 1e-10
    max_iters: int = 100_000
    precond: PrecondSpec = field(default_factory=PrecondSpec)
    precond_fp32: bool = False
    rcm: bool = False
    rhs: RhsSpec = field(default_factory=lambda: RhsSpec(RhsKind.ONES))
    switch_iter: int = 0
    seed: int = 0
    out: str | None = None
    allow_fp32_tol: bool = False

    def validate(self) -> "RunConfig":
        if (self.matrix is None) == (self.gen is None):
            raise ConfigError("exactly one of matrix= or gen= is required")
        if self.m < 1:
            raise ConfigError("m must be positive")
        if not 0.0 < self.rtol < 1.0:
            raise ConfigError("rtol must be in (0, 1)")
        if self.solver is SolverKind.FD and self.switch_iter % self.m != 0:
            raise ConfigError(f"switch_iter={self.switch_iter} is not a multiple of m={self.m}")
        if self.solver is SolverKind.SINGLE and self.rtol < FP32_RTOL_FLOOR and not self.allow_fp32_tol:
            raise ConfigError(f"an fp32 solve cannot target rtol={self.rtol:g} "
                              f"(floor ~{FP32_RTOL_FLOOR:g}); set allow_fp32_tol=true to override")
        return self


_CONFIG_KEYS = ("matrix", "gen", "solver", "m", "rtol", "max_iters", "precond", "precond_fp32", "rcm",
                "rhs", "switch_iter", "seed", "out", "allow_fp32_tol")
_BOOL = {"true": True, "1": True, "yes": True, "false": False, "0": False, "no": False}


def _parse_bool(text: str) -> bool:
    try:
        return _BOOL[text.strip().lower()]
    except KeyError:
        raise ConfigError(f"expected a boolean, got {text!r}") from None


def parse_run_config(text: str) -> RunConfig:
    """The ``key = value`` grammar (io.py:288-327): ``#`` comments, one key per
    line, unknown or duplicate keys rejected; returns a validated config."""
    values: dict[str, str] = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, eq, value = line.partition("=")
        key, value = key.strip().lower(), value.strip()
        if not eq:
            raise ConfigError(f"line {lineno}: expected key = value, got {raw!r}")
        if key not in _CONFIG_KEYS:
            raise ConfigError(f"line {lineno}: unknown key {key!r}")
        if key in values:
            raise ConfigError(f"line {lineno}: duplicate key {key!r}")
        values[key] = value
    if not values.get("solver"):
        raise ConfigError("solver required")
    try:
        solver = SolverKind(values["solver"].lower())
    except ValueError:
        raise ConfigError(f"unknown solver {values['solver']!r}; expected double|single|ir|fd") from None
    seed = int(values.get("seed", "0"))
    cfg = RunConfig(
        solver=solver,
        matrix=values.get("matrix") or None,
        gen=parse_stencil_spec(values["gen"]) if values.get("gen") else None,
        m=int(values.get("m", "50")),
        rtol=float(values.get("rtol", "1e-10")),
        max_iters=int(values.get("max_iters", "100000")),
        precond=PrecondSpec.parse(values.get("precond", "none")),
        precond_fp32=_parse_bool(values.get("precond_fp32", "false")),
        rcm=_parse_bool(values.get("rcm", "false")),
        rhs=parse_rhs_spec(values.get("rhs", "ones"), seed),
        switch_iter=int(values.get("switch_iter", "0")),
        seed=seed,
        out=values.get("out") or None,
        allow_fp32_tol=_parse_bool(values.get("allow_fp32_tol", "false")),
    )
    return cfg.validate()


def format_run_config(cfg: RunConfig) -> str:
    """Serialise so that ``parse_run_config(format_run_config(c)) == c`` (io.py:338-363)."""
    lines = [f"solver = {cfg.solver.value}"]
    if cfg.matrix:
        lines.append(f"matrix = {cfg.matrix}")
    if cfg.gen:
        kind = cfg.gen.kind.value
        extra = ""
        if kind in ("convdiff2d", "recirc2d"):
            extra = f":convection={cfg.gen.convection!r}"
        elif kind == "stretched2d":
            extra = f":stretch={cfg.gen.stretch!r}"
        lines.append(f"gen = {kind}:{cfg.gen.nx}{extra}")
    lines += [f"m = {cfg.m}", f"rtol = {cfg.rtol!r}", f"max_iters = {cfg.max_iters}",
              f"precond = {cfg.precond}", f"precond_fp32 = {str(cfg.precond_fp32).lower()}",
              f"rcm = {str(cfg.rcm).lower()}"]
    if cfg.rhs.kind is RhsKind.FROM_FILE:
        lines.append(f"rhs = file:{cfg.rhs.path}")
    else:
        lines.append(f"rhs = {cfg.rhs.kind.value}")
    lines += [f"switch_iter = {cfg.switch_iter}", f"seed = {cfg.seed}"]
    if cfg.out:
        lines.append(f"out = {cfg.out}")
    if cfg.allow_fp32_tol:
        lines.append("allow_fp32_tol = true")
    return "\n".join(lines) + "\n"


def load_run_config(path) -> RunConfig:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_run_config(fh.read())

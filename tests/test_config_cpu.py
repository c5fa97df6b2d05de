"""Run-configuration grammar and CLI argument handling (host only, no GPU).

Mirrors the reference's tests of io.parse_run_config / format_run_config and
cli._config_from_args; where the reference package is importable (the build
container) the two parsers are run on the same texts and must agree.
"""

import pytest

import paper_2109_01232_b200 as P
from paper_2109_01232_b200 import cli
from paper_2109_01232_b200.config import ConfigError, PrecondSpec, RunConfig, SolverKind

TEXTS = [
    "solver = ir\ngen = laplace3d:150\n",
    "solver = fd\ngen = laplace2d:100\nswitch_iter = 200\nm = 50  # comment\n",
    "solver = double\ngen = convdiff2d:1500:convection=1501.0\nprecond = jacobi:1\nprecond_fp32 = true\n",
    "solver = ir\ngen = laplace3d:200\nprecond = poly:25\nrtol = 1e-10\nseed = 7\nrhs = normal\n",
    "solver = single\ngen = laplace2d:50\nrtol = 1e-7\nallow_fp32_tol = yes\nmax_iters = 500\n",
    "solver = double\nmatrix = some/file.mtx\nrcm = true\nout = /tmp/x\n",
]

BAD = [
    "gen = laplace2d:50\n",                                  # solver required
    "solver = quad\ngen = laplace2d:50\n",                   # unknown solver
    "solver = ir\n",                                         # neither matrix nor gen
    "solver = ir\ngen = laplace2d:50\nmatrix = a.mtx\n",     # both
    "solver = fd\ngen = laplace2d:50\nswitch_iter = 75\n",   # not a multiple of m
    "solver = single\ngen = laplace2d:50\n",                 # fp32 cannot reach 1e-10
    "solver = ir\ngen = laplace2d:50\nbogus = 1\n",          # unknown key
    "solver = ir\nsolver = ir\ngen = laplace2d:50\n",        # duplicate key
    "solver = ir\ngen = laplace2d:50\nrtol = 2\n",           # rtol out of range
    "solver = ir\ngen = laplace2d:50\nprecond = ilu:1\n",    # unknown preconditioner
    "solver = ir\ngen = laplace2d:50\nrcm = maybe\n",        # not a boolean
    "solver ir\n",                                           # no '='
]


@pytest.mark.parametrize("text", TEXTS)
def test_round_trip(text):
    cfg = P.parse_run_config(text)
    again = P.parse_run_config(P.format_run_config(cfg))
    assert again == cfg


@pytest.mark.parametrize("text", BAD)
def test_rejections(text):
    with pytest.raises(ConfigError):
        P.parse_run_config(text)


@pytest.mark.parametrize("text", TEXTS + BAD)
def test_agrees_with_the_reference_parser(text, reference):
    from mpgmres import io as rio
    try:
        ref = rio.parse_run_config(text)
    except rio.ConfigError:
        with pytest.raises(ConfigError):
            P.parse_run_config(text)
        return
    ours = P.parse_run_config(text)
    assert P.format_run_config(ours) == rio.format_run_config(ref)


def test_precond_spec():
    assert PrecondSpec.parse("none") == PrecondSpec()
    assert PrecondSpec.parse("Poly:40") == PrecondSpec("poly", 40)
    assert str(PrecondSpec.parse("jacobi:4")) == "jacobi:4"
    for bad in ("jacobi:0", "poly:-1", "jacobi", "ilu:2"):
        with pytest.raises(ConfigError):
            PrecondSpec.parse(bad)


def test_cli_flags_override_the_config_file(tmp_path):
    f = tmp_path / "run.cfg"
    f.write_text("solver = double\ngen = laplace2d:50\nm = 30\nseed = 3\n")
    args = cli.build_parser().parse_args(["solve", "--config", str(f), "--solver", "ir", "--m", "40",
                                          "--precond", "poly:5", "--rhs", "normal"])
    cfg = cli.config_from_args(args)
    assert cfg.solver is SolverKind.IR and cfg.m == 40 and cfg.precond == PrecondSpec("poly", 5)
    assert cfg.rhs.kind.value == "normal" and cfg.rhs.seed == 3 and cfg.gen.nx == 50
    args = cli.build_parser().parse_args(["sweep-switch", "--gen", "laplace2d:20", "--solver", "fd",
                                          "--points", "0,50,100"])
    assert cli.config_from_args(args).gen.nx == 20 and cli._ints(args.points) == [0, 50, 100]


def test_cli_reports_bad_configs_with_exit_code_2(capsys):
    assert cli.main(["solve", "--gen", "laplace2d:50"]) == 2
    assert "solver required" in capsys.readouterr().err
    assert cli.main(["solve", "--solver", "fd", "--gen", "laplace2d:50", "--switch-iter", "7"]) == 2


def test_runconfig_defaults_match_the_reference():
    cfg = RunConfig(solver=SolverKind.IR, gen=P.parse_stencil_spec("laplace2d:10"))
    assert (cfg.m, cfg.rtol, cfg.max_iters, cfg.switch_iter, cfg.seed) == (50, 1e-10, 100_000, 0, 0)
    assert cfg.validate() is cfg

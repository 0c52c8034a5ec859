"""Expression templates on the host side: parser, validator, printer, model
files (mirroring /root/reference/pkg/tests/test_dsl.py), CUDA code generation
and NVRTC compilation of the generated programs (no GPU needed)."""

import numpy as np
import pytest

import paper_1908_03869_b200 as sdb
from paper_1908_03869_b200 import dsl, program
from paper_1908_03869_b200.model import KURAMOTO_DIFFUSION_TEMPLATE, KURAMOTO_DRIFT_TEMPLATE


def _shape(node):
    return dsl.strip_positions(node)


# ---- parsing (test_dsl.py:24-86) -------------------------------------------------

@pytest.mark.parametrize("src, want", [
    ("2+3*4", dsl.BinOp("+", dsl.Num(2.0), dsl.BinOp("*", dsl.Num(3.0), dsl.Num(4.0)))),
    ("2^3^2", dsl.BinOp("^", dsl.Num(2.0), dsl.BinOp("^", dsl.Num(3.0), dsl.Num(2.0)))),
    ("-2^2", dsl.Neg(dsl.BinOp("^", dsl.Num(2.0), dsl.Num(2.0)))),
    ("2^-1", dsl.BinOp("^", dsl.Num(2.0), dsl.Neg(dsl.Num(1.0)))),
    ("8/4/2", dsl.BinOp("/", dsl.BinOp("/", dsl.Num(8.0), dsl.Num(4.0)), dsl.Num(2.0))),
    ("--2", dsl.Neg(dsl.Neg(dsl.Num(2.0)))),
    ("-a*b", dsl.BinOp("*", dsl.Neg(dsl.Var("a")), dsl.Var("b"))),
])
def test_precedence_and_associativity(src, want):
    assert _shape(dsl.parse(src)) == want


def test_parse_sum_node():
    node = dsl.parse("sum(j, sin(y[j]-y[i]))")
    assert isinstance(node, dsl.Sum) and node.var == "j" and isinstance(node.body, dsl.Call)


@pytest.mark.parametrize("source", ["2+", "sin(", "(1+2", "y[", "y[0", "sum(j y[j])",
                                    "sum(, 1)", "1 2"])
def test_syntax_errors(source):
    with pytest.raises(dsl.ParseError):
        dsl.parse(source)


def test_error_kinds_and_positions():
    with pytest.raises(dsl.ParseError, match="unknown function"):
        dsl.parse("sinh(1)")
    with pytest.raises(dsl.ParseError, match="can be indexed"):
        dsl.parse("q[0]")
    with pytest.raises(dsl.ParseError, match="index name"):
        dsl.parse("sum(1, 2)")
    with pytest.raises(dsl.ParseError) as err:
        dsl.parse("1 +\n 2 $ 3")
    assert (err.value.line, err.value.col) == (2, 4)


# ---- validation (test_dsl.py:92-132) ----------------------------------------------

def test_validation_diagnostics():
    assert "out of range" in dsl.validate(dsl.parse("y[5]"), 5, 0, 0)[0].message
    assert any("drift" in d.message
               for d in dsl.validate(dsl.parse("n[0]"), 1, 0, 1, role="drift"))
    assert dsl.validate(dsl.parse("n[0]"), 1, 0, 1, role="diffusion") == []
    n = 100
    assert dsl.validate(dsl.parse(KURAMOTO_DRIFT_TEMPLATE), n, 2 * n + 1, n, role="drift") == []
    assert dsl.validate(dsl.parse(KURAMOTO_DIFFUSION_TEMPLATE), n, 2 * n + 1, n) == []
    assert any("nested sums" in d.message
               for d in dsl.validate(dsl.parse("sum(j, sum(j, y[j]))"), 3, 0, 0))
    assert dsl.validate(dsl.parse("sum(j, sum(k, y[j]*y[k]))"), 3, 0, 0) == []
    assert any("unknown variable" in d.message for d in dsl.validate(dsl.parse("z + 1"), 1, 0, 0))
    assert any("reserved" in d.message for d in dsl.validate(dsl.parse("sum(i, y[i])"), 3, 0, 0))
    for src in ["y[0.5]", "y[t]", "y[i/2]", "y[sqrt(4)]"]:
        assert dsl.validate(dsl.parse(src), 4, 0, 0) != []
    with pytest.raises(ValueError):
        dsl.validate(dsl.parse("1"), 1, 0, 0, role="other")


def test_model_from_dsl_validates():
    with pytest.raises(sdb.ModelDefinitionError, match="invalid model"):
        sdb.model_from_dsl("bad", nequat=2, nparams=1, nnoise=2, drift="p[3]", diffusion="n[0]")
    with pytest.raises(sdb.ModelDefinitionError, match="drift"):
        sdb.model_from_dsl("bad", nequat=2, nparams=1, nnoise=2, drift="n[0]", diffusion="0")


# ---- printer round trip (test_dsl.py:231-250) ---------------------------------------

ROUND_TRIP = ["2+3*4", "-(y[0]+p[0])", "-y[0]^2", "(2+3)*(4-1)", "2^3^2", "(2^3)^2", "8/4/2",
              "8/(4/2)", "1 - 2 - 3", "1 - (2 - 3)", KURAMOTO_DRIFT_TEMPLATE,
              "sum(j, sum(k, cos(y[j]-y[k])))/N", "exp(0-t)*sqrt(abs(y[0]))",
              KURAMOTO_DIFFUSION_TEMPLATE, "2^-3^2", "-(2)^-(1)", "a - -b"]


@pytest.mark.parametrize("source", ROUND_TRIP)
def test_print_parse_round_trip_is_structural(source):
    node = dsl.parse(source)
    assert _shape(dsl.parse(dsl.to_source(node))) == _shape(node)


# ---- model files (test_dsl.py:256-290) ------------------------------------------------

MODEL_TEXT = """
# a linear system with additive noise
nequat=2
nparams=3
nnoise=2

drift: 0 - p[0]*y[i]
diffusion: p[1+i]*n[i]
"""


def test_model_text_and_files(tmp_path):
    c = dsl.parse_model_text(MODEL_TEXT, name="linear")
    assert (c.nequat, c.nparams, c.nnoise, c.name) == (2, 3, 2, "linear")
    assert c.drift.startswith("0 - ")
    with pytest.raises(dsl.ParseError, match="missing header"):
        dsl.parse_model_text("drift: 1\ndiffusion: 0\n")
    with pytest.raises(dsl.ParseError, match="missing 'diffusion'"):
        dsl.parse_model_text("nequat=1\nnparams=0\nnnoise=0\ndrift: 1\n")
    with pytest.raises(dsl.ParseError, match="duplicate"):
        dsl.parse_model_text("nequat=1\nnequat=2\nnparams=0\nnnoise=0\ndrift: 1\ndiffusion: 0\n")
    with pytest.raises(dsl.ParseError, match="unrecognised"):
        dsl.parse_model_text("nequat=1\nwhat is this\n")
    path = tmp_path / "linear.model"
    path.write_text(MODEL_TEXT, encoding="utf-8")
    m = sdb.model_from_file(path)
    assert (m.name, m.nequat, m.nnoise) == ("linear", 2, 2)
    assert sdb.model.expression_model(m)


# ---- recognition and index checks ------------------------------------------------------

def test_kuramoto_templates_use_the_native_stepper(monkeypatch):
    m = sdb.kuramoto_dsl_model(6)
    assert sdb.model.kuramoto_signature(m) == (6, 6)
    assert not sdb.model.expression_model(m)
    monkeypatch.setenv("SDEB200_NO_NATIVE_KURAMOTO", "1")
    assert sdb.model.kuramoto_signature(m) is None and sdb.model.expression_model(m)


def test_index_checks():
    program.check_indices(dsl.parse("y[i] + sum(j, p[j + i])"), 3, {"y": 3, "p": 5}, range(3))
    with pytest.raises(dsl.DomainError, match="out of range"):
        program.check_indices(dsl.parse("sum(j, p[j + i])"), 3, {"y": 3, "p": 4}, range(3))
    with pytest.raises(dsl.DomainError, match="out of range"):
        program.check_indices(dsl.parse("y[i+1]"), 3, {"y": 3}, range(3))
    program.check_indices(dsl.parse("y[i+1]"), 3, {"y": 3}, [0, 1])
    with pytest.raises(dsl.DomainError, match="not available"):
        program.check_indices(dsl.parse("n[0]"), 3, {"y": 3}, range(3))
    nested = dsl.parse("sum(j, sum(k, y[j] * p[k * 3 + j]))")
    program.check_indices(nested, 3, {"y": 3, "p": 9}, range(3))
    with pytest.raises(dsl.DomainError):
        program.check_indices(nested, 3, {"y": 3, "p": 8}, range(3))
    bad = sdb.model_from_dsl("shift", 3, 0, 0, "y[i+1]", "0")
    with pytest.raises(dsl.DomainError):
        sdb.run_batch(bad, sdb.EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=1),
                      sdb.OrbitBatch(init=np.zeros((1, 3)), params=np.zeros((1, 0))))


# ---- code generation + NVRTC (host only) ----------------------------------------------

def test_generated_code_follows_the_templates():
    cm = program.compiled(4, 9, 4, dsl.parse(KURAMOTO_DRIFT_TEMPLATE),
                          dsl.parse(KURAMOTO_DIFFUSION_TEMPLATE))
    src = cm.source(0)
    assert "#define SDB_N 4" in src and "#define SDB_KIND 0" in src
    assert "dsl_sum(" in src and "dsl_sin<EXACT>(__dsub_rn(y[s_j], y[i]), big)" in src
    assert "__ddiv_rn(p[0], kDslN)" in src
    assert "__dmul_rn(p[((1 + SDB_N) + i)], n[i])" in src


def test_bad_templates_fail_in_codegen():
    with pytest.raises(ValueError, match="drift: line 1"):
        program.CompiledModel(2, 1, 0, "y[0] +* 1", "0")
    with pytest.raises(ValueError, match="unknown function"):
        program.CompiledModel(2, 1, 0, "foo(1)", "0")
    with pytest.raises(ValueError, match="drift"):
        program.CompiledModel(2, 1, 1, "n[0]", "0")


@pytest.mark.parametrize("kind", [0, 1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_programs_compile_with_nvrtc(kind):
    # every program kind of a model exercising all grammar features compiles
    # for sm_100a (NVRTC needs no GPU)
    cm = program.compiled(
        3, 5, 3,
        dsl.parse("-(y[i]^3) + sin(t) * p[i] + sum(j, sum(k, y[j]*p[k]/(1 + abs(y[k])))) "
                  "- 2^-3^2 + cos(y[i]) * tan(0.1*t) / N"),
        dsl.parse("sqrt(abs(y[i])) * n[i] + exp(-t) * ln(1 + y[i]*y[i]) + p[4] * n[2 - i]"))
    cm.build(kind)


def test_lane_groups_and_state_placement(monkeypatch):
    small = program.compiled(3, 1, 3, dsl.parse("p[0] - y[i]"), dsl.parse("n[i]"))
    assert "#define SDB_LANES 1" in small.source(0)
    mid = program.compiled(16, 1, 16, dsl.parse("p[0] - y[i]"), dsl.parse("n[i]"))
    assert "#define SDB_LANES 1" in mid.source(0)  # O(1) per equation: one lane
    mid_sum = program.compiled(16, 1, 16, dsl.parse("p[0] - sum(j, y[j] * y[i])"),
                               dsl.parse("n[i]"))
    assert "#define SDB_LANES 4" in mid_sum.source(0)  # O(N) per equation: ~4 per lane
    hoisted = program.compiled(16, 1, 16, dsl.parse("p[0] - sum(j, y[j])"), dsl.parse("n[i]"))
    assert "#define SDB_LANES 1" in hoisted.source(0)  # the sum is computed once per step
    big = program.compiled(400, 1, 400, dsl.parse("p[0] - sum(j, y[j] - y[i])"),
                           dsl.parse("n[i]"))
    src = big.source(0)
    assert "#define SDB_LANES 32" in src and "#define SDB_GLOBAL_STATE 0" in src
    # one lane per orbit: 128 columns of 800 doubles exceed shared memory
    monkeypatch.setenv("SDEB200_DSL_LANES", "1")
    src = big.source(0)
    assert "#define SDB_LANES 1" in src and "#define SDB_GLOBAL_STATE 1" in src
    big.build(0)


def test_factored_and_hoisted_code():
    cm = program.compiled(8, 17, 8, dsl.parse(KURAMOTO_DRIFT_TEMPLATE),
                          dsl.parse(KURAMOTO_DIFFUSION_TEMPLATE))
    lit, fac = cm.source(0), cm.source(0, factored=True)
    # literal: the n^2 sin terms as written; factored: one sincos pass over j,
    # hoisted into the prologue, combined per equation by the addition formula
    assert "dsl_sin<EXACT>(__dsub_rn(y[s_j], y[i]), big)" in lit and "dsl_sum_sincos" not in lit
    # the equation's angle y[i] is the j-term at j = i: the pass keeps every term's
    # (sin, cos) for the equations instead of a second sincos each
    assert ("dsl_sum_sincos_keep<EXACT>([&](int s_j) -> double { return y[s_j]; }, big, H[0], "
            "H[1], &H[2], &H[2 + SDB_N]);") in fac
    assert "H[2 + SDB_N + i]" in fac and "dsl_cos<EXACT>" not in fac.split("sdb_drift(int i")[1]
    assert "#define SDB_DRIFT_H %d" % (2 + 2 * 8) in fac and "#define SDB_DRIFT_H 1" in lit
    # a different equation-side angle: a second sincos per equation
    other = program.compiled(4, 1, 0, dsl.parse("sum(j, cos(y[j] - 2 * y[i]))"), None)
    assert "dsl_sum_sincos<EXACT>" in other.source(3, factored=True)
    # equation-independent sums are hoisted in both forms (bit-identical)
    m = program.compiled(3, 1, 0, dsl.parse("p[0] * sum(j, y[j]) - y[i]"), None)
    for form in (m.source(3), m.source(3, factored=True)):
        assert "H[0] = dsl_sum([&](int s_j) -> double { return y[s_j]; });" in form
        assert "__dmul_rn(p[0], H[0])" in form
    # sums that read i stay per equation; sin(A - B) with both sides reading j is not factored
    k = program.compiled(3, 1, 0, dsl.parse("sum(j, sin(y[j] - y[j] * y[i])) + sum(j, y[j] * i)"),
                         None)
    assert "H[0]" not in k.source(3, factored=True).split("sdb_drift(int i")[1]
    for kind in (0, 3, 4, 8):
        cm.build(kind, factored=True)

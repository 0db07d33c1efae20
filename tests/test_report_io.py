"""CPU: the report formats and the OCPROB01 container are byte-compatible with
the reference (report_io.cpp, problems.cpp:327-416).  The golden text was
written by the reference itself (oracle/make_golden.py)."""
import io
import os
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1810_03930_b200 import report_io as R

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _report_from_reference_json(text):
    d = R.run_report_from_json(text)
    fin = lambda f: None if f is None else SimpleNamespace(**f)
    return SimpleNamespace(trace=d["trace"], final_pre_orth=fin(d["final_pre_orth"]),
                           final_post_orth=fin(d["final_post_orth"]), iterations=d["iterations"],
                           degenerate_steps=d["degenerate_steps"], status=d["status"],
                           wall_time=d["wall_time"], stop_iterate=None, final_x=None), d


def test_json_report_byte_identical_to_reference():
    ref_text = open(os.path.join(GOLD, "ref_report_p1_n60.json")).read()
    rep, d = _report_from_reference_json(ref_text)
    assert R.to_json(rep, d["config"]) + "\n" == ref_text


def test_json_number_format_matches_nlohmann_at_every_magnitude():
    """nlohmann's dtoa switches to exponent form above 15 integer digits
    (1e15 ≤ |v| < 1e16 is "1e+15", Python's repr says "1000000000000000.0"):
    the reference's own to_json of a report holding those values, byte for byte
    (ref_report_magnitudes.json, oracle/make_golden.py json_magnitudes_case)."""
    ref_text = open(os.path.join(GOLD, "ref_report_magnitudes.json")).read()
    assert '"fval": 1e+15,' in ref_text and '1.5e+15' in ref_text
    rep, d = _report_from_reference_json(ref_text)
    assert R.to_json(rep, d["config"]) + "\n" == ref_text


def test_trace_csv_byte_identical_to_reference():
    ref_text = open(os.path.join(GOLD, "ref_trace_p1_n60.csv")).read()
    rep, _ = _report_from_reference_json(open(os.path.join(GOLD, "ref_report_p1_n60.json")).read())
    out = io.StringIO()
    R.write_trace_csv(rep, out)
    assert out.getvalue() == ref_text


def test_summary_row_and_same_numerics():
    rep, d = _report_from_reference_json(open(os.path.join(GOLD, "ref_report_p1_n60.json")).read())
    out = io.StringIO()
    R.write_summary_header(out)
    R.write_summary_row(rep, d["config"], out)
    lines = out.getvalue().splitlines()
    assert lines[1].startswith("p1,pcal,7,60,4,1,abb,max-iter,50,0,")
    assert R.same_numerics(rep, rep)
    other = SimpleNamespace(**vars(rep))
    other.trace = rep.trace.copy()
    other.trace[3, 1] = np.nextafter(other.trace[3, 1], 0)
    assert not R.same_numerics(rep, other)


def test_container_round_trip_byte_identical(pcal):
    path = os.path.join(GOLD, "ref_quad40.ocprob")
    ref = np.load(os.path.join(GOLD, "ref_quad40.npz"))
    model, params = R.load_problem(path, pcal)
    assert params["tag"] == 2 and model.n == 40 and model.p == 5 and model.s == float(ref["s"])
    assert np.array_equal(model.a, ref["a"]) and np.array_equal(model.g0, ref["g0"])
    out = io.BytesIO()
    R.save_problem(model, out, **{k: params[k] for k in ("kappa", "theta", "zeta", "xi")})
    assert out.getvalue() == open(path, "rb").read()


def test_harness_problem_spec_checks_are_host_side():
    """make_problem's parameter checks (problems.cpp gen_problem*, harness.cpp:31-46)
    and the kinds without a device model fail before any device work."""
    from paper_1810_03930_b200 import harness as H
    from paper_1810_03930_b200.report_io import UnsupportedModel
    with pytest.raises(pcal_errors().ParameterError):
        H.make_problem(H.ProblemSpec(kind="p1", n=10, p=6, alpha=0.0))      # 2p > n
    with pytest.raises(UnsupportedModel):
        H.make_problem(H.ProblemSpec(kind="p5", n=40, p=4))                 # no such kind
    with pytest.raises(pcal_errors().ParameterError):
        H.make_problem(H.ProblemSpec(kind="p1", n=40, p=4, alpha=-1.0))
    with pytest.raises(pcal_errors().ParameterError):
        H.make_problem(H.ProblemSpec(kind="p1", n=42, p=4, alpha=0.0, mode="block-tridiag"))
    with pytest.raises(pcal_errors().ParameterError):
        H.make_problem(H.ProblemSpec(kind="p2", n=40, p=4, theta=0.5))


def test_density_inverse_is_the_reference_linear_solver():
    """pcal_density_inverse = LinearSolver (linsolve.cpp:30-102) against e_c, bitwise,
    on both factorisation paths; a singular L is the reference's generation_error."""
    import paper_1810_03930_b200 as P
    g = np.load(os.path.join(GOLD, "reference_linsolve.npz"))
    for name in ("lu", "chol"):
        assert not bool(g[name + "_singular"])
        assert np.array_equal(P.density_inverse(g[name + "_a"]), g[name + "_inv"])
    assert bool(g["singular_singular"])
    with pytest.raises(P.ParameterError):
        P.density_inverse(g["singular_a"])


@pytest.mark.parametrize("name,spec", [
    ("p1_alpha1", dict(kind="p1", n=80, p=5, alpha=1.0, seed=21)),
    ("p1_block_alpha2", dict(kind="p1", n=60, p=4, alpha=2.0, mode="block-tridiag", seed=22)),
    ("p4", dict(kind="p4", n=60, p=5, seed=23)),
    ("p6", dict(kind="p6", n=70, p=4, seed=24)),
])
def test_harness_instances_match_reference(name, spec):
    """gen_problem1 (α > 0) / gen_problem4 / gen_problem6 on the host: the curvature
    scale the reference echoes in its own run_single report, bitwise."""
    import json
    from paper_1810_03930_b200 import harness as H
    ref = json.load(open(os.path.join(GOLD, f"ref_run_single_{name}.json")))
    m = H.make_problem(H.ProblemSpec(**spec))
    assert m.s == ref["config"]["curvature_scale"]
    assert m.n == spec["n"] and m.p == spec["p"]


def test_host_spectral_norm_is_the_reference_one():
    """spectral_norm_estimate (kernels.cpp:267-293): the host version is bitwise the
    reference's (golden value of the reference's own run, and config 1's s)."""
    import paper_1810_03930_b200 as P
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_small.npz"))
    assert P.spectral_norm_estimate_host(g["k_spec_a"], 11) == float(g["k_spec_s"])
    assert P.spectral_norm_estimate_host(P.gen_dense_operator(1000, 1), 1 ^ 0x73706563) == \
        float(g["cfg1_s"])


def pcal_errors():
    import paper_1810_03930_b200 as P
    return P


def test_run_matrix_records_failed_cells_without_a_gpu():
    """run_matrix (harness.cpp:75-104): a cell whose generation fails is a
    'diverged' summary row (echo of the cell, no numbers) and never aborts the
    matrix — byte-identical to the reference's rows for the same cells."""
    import io as _io
    from paper_1810_03930_b200 import harness as H
    import paper_1810_03930_b200 as P
    with pytest.raises(P.ParameterError):
        H.run_matrix(H.MatrixSpec(problems=[], solvers=["pcal"], seeds=[1]), _io.StringIO())
    out = _io.StringIO()
    H.run_matrix(H.MatrixSpec(problems=[H.ProblemSpec(kind="p1", n=32, p=3, mode="block-tridiag")],
                              solvers=["pcal", "plam", "alm"], seeds=[1, 2],
                              base=P.SolverConfig(max_iter=500)), out)
    ref = open(os.path.join(GOLD, "ref_matrix.csv")).read().splitlines()
    assert out.getvalue().splitlines() == [ref[0]] + ref[-6:]


@pytest.mark.parametrize("name,spec", [
    ("p4", dict(kind="p4", n=12, p=3, seed=41)),
    ("p1", dict(kind="p1", n=10, p=2, alpha=1.5, mode="block-tridiag", seed=42)),
    ("p6", dict(kind="p6", n=11, p=3, seed=43)),
])
def test_bilinear_density_containers_match_reference(name, spec):
    """save_problem of the Bilinear / Density models (problems.cpp:341-361):
    the harness's instance saves to the reference's container byte for byte,
    and load_problem rebuilds the same model."""
    import io as _io
    from paper_1810_03930_b200 import harness as H
    from paper_1810_03930_b200 import report_io as R
    path = os.path.join(GOLD, f"ref_{name}.ocprob")
    m = H.make_problem(H.ProblemSpec(**spec))
    out = _io.BytesIO()
    R.save_problem(m, out)
    assert out.getvalue() == open(path, "rb").read()
    back, params = R.load_problem(path)
    assert back.kind == m.kind and (back.n, back.p, back.s) == (m.n, m.p, m.s)
    assert np.array_equal(back.a, m.a)
    if name == "p4":
        assert np.array_equal(back.b, m.b)
    else:
        assert back.coeff == m.coeff and back.variant == m.variant and back.mode == m.mode
        assert np.array_equal(back.linv, m.linv)

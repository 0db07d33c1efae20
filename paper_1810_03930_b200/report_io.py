"""Run-report emission and the problem container of the reference.

* ``to_json`` / ``run_report_from_json`` — the reference's JSON run report
  (report_io.cpp:86-136): same keys, key order (nlohmann's sorted map), 2-space
  indentation and shortest round-trip number formatting, so a report of the
  same numbers is byte-identical to the reference's ``write_report_file``.
* ``write_trace_csv`` — ``iter,fval,kkt_abs,kkt_rel,feas,eta,time_ms`` with
  ``%.17g`` (report_io.cpp:165-172); ``write_summary_header`` / ``_row``
  (report_io.cpp:174-194); ``same_numerics`` (report_io.cpp:259-283).
* ``save_problem`` / ``load_problem`` — the ``OCPROB01`` binary container
  (problems.cpp:327-416) for every reference family: the dense quadratic
  (tags 2, 3), P4 bilinear (4) and the P1 / P6 density models (1, 6).  Only the
  models the reference has no container for (grid, Kohn–Sham, caller-defined)
  raise ``UnsupportedModel``.
"""
from __future__ import annotations

import io
import json
import math
import struct
from dataclasses import asdict, dataclass
from typing import IO, Optional

import numpy as np

MAGIC = b"OCPROB01"
STATUS_TEXT = {"converged": "converged", "max_iter": "max-iter", "diverged": "diverged"}
STATUS_FROM_TEXT = {"converged": "converged", "max-iter": "max_iter", "diverged": "diverged"}


class UnsupportedModel(ValueError):
    """The container holds a model family without a device evaluator."""


@dataclass
class ConfigEcho:
    """ConfigEcho (report.hpp:22-36)."""
    problem: str = "p3"
    n: int = 0
    p: int = 0
    solver: str = "pcal"
    beta: float = 0.0
    eta_rule: str = "abb"
    tol_rel_kkt: float = 1e-8
    max_iter: int = 0
    threads: int = 1
    init: str = "qr"
    seed: int = 0
    alpha: float = 0.0
    kappa: float = 0.0
    theta: float = 0.0
    zeta: float = 0.0
    xi: float = 0.0
    curvature_scale: float = 0.0


ETA_RULE_NAMES = {0: None, 1: "diff", 2: "bb1", 3: "bb2", 4: "abb"}


def eta_rule_name(rule) -> str:
    """eta_rule_name (solver.cpp:41-50)."""
    if rule.kind == 0:
        return "const:" + f"{rule.gamma:.6f}"  # std::to_string(double)
    return ETA_RULE_NAMES[rule.kind]


def echo_for(model, config, report, problem: str = "p3", seed: int = 0, init: str = "qr",
             threads: int = 1, **params) -> ConfigEcho:
    """The echo iterate_main + fill_config_echo write (solver.cpp:332-342, harness.cpp:48-60)."""
    return ConfigEcho(problem=problem, n=model.n, p=model.p, solver=config.algorithm,
                      beta=report.beta, eta_rule=eta_rule_name(config.eta_rule),
                      tol_rel_kkt=config.tol_rel_kkt, max_iter=config.max_iter, threads=threads,
                      init=init, seed=seed, curvature_scale=model.s, **params)


def _num(v):
    if isinstance(v, float) and not math.isfinite(v):
        return None  # nlohmann writes non-finite doubles as null
    return v


def _nl_double(v: float) -> str:
    """A finite double as nlohmann::json writes it (dtoa_impl::format_buffer with
    min_exp = −4, max_exp = digits10 = 15): the shortest round-trip digits D
    with v = 0.D·10ⁿ, positional for −4 < n ≤ 15 (integers get ".0"),
    exponent form otherwise ("1e+15", "1.5e-05": sign and ≥ 2 exponent digits).
    Python's repr differs exactly for 1e15 ≤ |v| < 1e16 (it stays positional
    up to n = 16)."""
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    r = repr(v)
    sign = "-" if r[0] == "-" else ""
    r = r.lstrip("-")
    mant, _, e = r.partition("e")
    ip, _, fp = mant.partition(".")
    digits = ip + fp
    n = len(ip) + (int(e) if e else 0)
    stripped = digits.lstrip("0")
    n -= len(digits) - len(stripped)
    d = stripped.rstrip("0")
    k = len(d)
    if k <= n <= 15:
        body = d + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        body = d[:n] + "." + d[n:]
    elif -4 < n <= 0:
        body = "0." + "0" * (-n) + d
    else:
        x = n - 1
        body = (d if k == 1 else d[0] + "." + d[1:]) + "e" + ("-" if x < 0 else "+") + \
            f"{abs(x):02d}"
    return sign + body


def _dumps(obj, level: int = 0) -> str:
    """json.dumps(obj, indent=2, sort_keys=True) with nlohmann's double format."""
    pad, inner = "  " * level, "  " * (level + 1)
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f"{inner}{json.dumps(str(k))}: {_dumps(obj[k], level + 1)}" for k in sorted(obj)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(obj, (list, tuple)):
        if not obj:
            return "[]"
        return "[\n" + ",\n".join(inner + _dumps(v, level + 1) for v in obj) + "\n" + pad + "]"
    if isinstance(obj, bool) or obj is None or isinstance(obj, (int, str)):
        return json.dumps(obj)
    if isinstance(obj, float):
        return _nl_double(obj) if math.isfinite(obj) else "null"
    raise TypeError(f"not JSON-serialisable: {type(obj).__name__}")


def _final(f) -> dict:
    return {"feas": _num(float(f.feas)), "fval": _num(float(f.fval)),
            "kkt_abs": _num(float(f.kkt_abs)), "kkt_rel": _num(float(f.kkt_rel))}


def to_json(report, echo: ConfigEcho, include_timing: bool = False,
            outer_iterations: Optional[int] = None, inner_cap_hits: Optional[int] = None) -> str:
    """to_json(RunReport) (report_io.cpp:86-106).  The ALM counters default to the
    report's own (0 for the other algorithms)."""
    if outer_iterations is None:
        outer_iterations = int(getattr(report, "outer_iterations", 0))
    if inner_cap_hits is None:
        inner_cap_hits = int(getattr(report, "inner_cap_hits", 0))
    cfg = {k: _num(v) for k, v in asdict(echo).items()}
    trace = []
    for row in report.trace:
        d = {"iter": int(row[0]), "fval": _num(float(row[1])), "kkt_abs": _num(float(row[2])),
             "kkt_rel": _num(float(row[3])), "feas": _num(float(row[4])), "eta": _num(float(row[5]))}
        if include_timing:
            d["elapsed"] = float(row[6])
        trace.append(d)
    j = {"config": cfg, "trace": trace, "final": {"pre_orth": _final(report.final_pre_orth)},
         "iterations": int(report.iterations), "outer_iterations": outer_iterations,
         "inner_cap_hits": inner_cap_hits, "degenerate_steps": int(report.degenerate_steps),
         "status": STATUS_TEXT[report.status]}
    if report.final_post_orth is not None:
        j["final"]["post_orth"] = _final(report.final_post_orth)
    if include_timing:
        j["wall_time"] = float(report.wall_time)
    return _dumps(j)


def run_report_from_json(text: str) -> dict:
    """run_report_from_json (report_io.cpp:108-136), as plain Python values."""
    j = json.loads(text)
    trace = np.array([[r["iter"], r["fval"], r["kkt_abs"], r["kkt_rel"], r["feas"], r["eta"],
                       r.get("elapsed", 0.0)] for r in j["trace"]], dtype=float).reshape(-1, 7)
    return {"config": ConfigEcho(**j["config"]), "trace": trace,
            "final_pre_orth": j["final"]["pre_orth"], "final_post_orth": j["final"].get("post_orth"),
            "iterations": j["iterations"], "outer_iterations": j["outer_iterations"],
            "inner_cap_hits": j["inner_cap_hits"], "degenerate_steps": j["degenerate_steps"],
            "wall_time": j.get("wall_time", 0.0), "status": STATUS_FROM_TEXT[j["status"]]}


def _g17(v: float) -> str:
    return "%.17g" % v


def write_trace_csv(report, out: IO[str]) -> None:
    """write_trace_csv (report_io.cpp:165-172)."""
    out.write("iter,fval,kkt_abs,kkt_rel,feas,eta,time_ms\n")
    for r in report.trace:
        out.write(f"{int(r[0])},{_g17(r[1])},{_g17(r[2])},{_g17(r[3])},{_g17(r[4])},{_g17(r[5])},"
                  f"{_g17(r[6] * 1000.0)}\n")


def write_summary_header(out: IO[str]) -> None:
    out.write("problem,solver,seed,n,p,beta,eta_rule,status,iterations,outer_iterations,"
              "fval,kkt_abs,kkt_rel,feas,fval_orth,kkt_abs_orth,kkt_rel_orth,feas_orth,"
              "time_s\n")


def write_summary_row(report, echo: ConfigEcho, out: IO[str],
                      outer_iterations: Optional[int] = None) -> None:
    """write_summary_row (report_io.cpp:181-194)."""
    if outer_iterations is None:
        outer_iterations = int(getattr(report, "outer_iterations", 0))
    f = report.final_pre_orth
    out.write(f"{echo.problem},{echo.solver},{echo.seed},{echo.n},{echo.p},{_g17(echo.beta)},"
              f"{echo.eta_rule},{STATUS_TEXT[report.status]},{report.iterations},"
              f"{outer_iterations},{_g17(f.fval)},{_g17(f.kkt_abs)},{_g17(f.kkt_rel)},"
              f"{_g17(f.feas)},")
    po = report.final_post_orth
    if po is not None:
        out.write(f"{_g17(po.fval)},{_g17(po.kkt_abs)},{_g17(po.kkt_rel)},{_g17(po.feas)}")
    else:
        out.write(",,,")
    out.write(f",{_g17(report.wall_time)}\n")


def same_numerics(a, b) -> bool:
    """same_numerics (report_io.cpp:259-283): bitwise equality of every number."""
    def beq(x, y):
        return np.array_equal(np.asarray(x, dtype=np.float64).view(np.uint64),
                              np.asarray(y, dtype=np.float64).view(np.uint64))
    if (a.status, a.iterations, a.degenerate_steps) != (b.status, b.iterations, b.degenerate_steps):
        return False
    if getattr(a, "outer_iterations", 0) != getattr(b, "outer_iterations", 0):
        return False
    if a.trace.shape != b.trace.shape or not beq(a.trace[:, :6], b.trace[:, :6]):
        return False
    for m1, m2 in ((a.stop_iterate, b.stop_iterate), (a.final_x, b.final_x)):
        if (m1 is None) != (m2 is None) or (m1 is not None and not beq(m1, m2)):
            return False
    fa, fb = a.final_pre_orth, b.final_pre_orth
    if not beq([fa.fval, fa.kkt_abs, fa.kkt_rel, fa.feas], [fb.fval, fb.kkt_abs, fb.kkt_rel, fb.feas]):
        return False
    pa, pb = a.final_post_orth, b.final_post_orth
    if (pa is None) != (pb is None):
        return False
    return pa is None or beq([pa.fval, pa.kkt_abs, pa.kkt_rel, pa.feas],
                             [pb.fval, pb.kkt_abs, pb.kkt_rel, pb.feas])


# ---- OCPROB01 container (problems.cpp:327-416) -----------------------------------
def _sym_upper(raw: bytes, n: int) -> np.ndarray:
    """get_symmetric (problems.cpp:93-99): the upper triangle mirrored."""
    a = np.frombuffer(raw, dtype="<f8").reshape((n, n), order="F").copy(order="F")
    iu = np.triu_indices(n)
    a[(iu[1], iu[0])] = a[iu]  # set_mirrored(i, j, upper(i, j))
    return a


def save_problem(model, out, kappa: float = 0.0, theta: float = 1.0, zeta: float = 1.0,
                 xi: float = 1.0) -> None:
    """save_problem (problems.cpp:327-366), little endian after the magic:
    QuadraticModel — u32 tag (2 with a linear term, 3 without), u64 n, u64 p,
    f64 s, kappa, theta, zeta, xi, A (n×n), G (n×p); BilinearModel — tag 4,
    n, p, s, A, B (p×p); DensityModel — tag 1 / 6, n, p, s, f64 coeff,
    u32 mode (1 = block-tridiagonal), L (n×n)."""
    kind = getattr(model, "kind", None)

    def head(tag):
        return MAGIC + struct.pack("<IQQd", tag, model.n, model.p, model.s)

    def mat(m):
        return np.asfortranarray(m, dtype="<f8").tobytes(order="F")
    if kind == 1:
        g = np.zeros((model.n, model.p), order="F") if model.g0 is None else model.g0
        buf = head(3 if model.g0 is None else 2) + struct.pack("<dddd", kappa, theta, zeta, xi)
        buf += mat(model.a) + mat(g)
    elif kind == 5:
        buf = head(4) + mat(model.a) + mat(model.b)
    elif kind == 6:
        buf = head(6 if model.variant == "p6" else 1)
        buf += struct.pack("<dI", model.coeff, 1 if model.mode == "block-tridiag" else 0)
        buf += mat(model.a)
    else:
        raise UnsupportedModel("save_problem: grid and callback models have no container form")
    if isinstance(out, (str, bytes)):
        with open(out, "wb") as f:
            f.write(buf)
    else:
        out.write(buf)


def load_problem(src, pcal=None):
    """load_problem (problems.cpp:368-416) → (model, params dict): QuadraticModel
    (tags 2 / 3), BilinearModel (4), DensityModel (1 / 6); symmetric matrices are
    symmetrised from their upper triangle like get_symmetric."""
    if pcal is None:
        import paper_1810_03930_b200 as pcal
    data = open(src, "rb").read() if isinstance(src, (str, bytes)) else src.read()
    f = io.BytesIO(data)
    if f.read(8) != MAGIC:
        raise ValueError("load_problem: bad magic bytes")
    tag, n, p, s = struct.unpack("<IQQd", f.read(28))

    def take(count):
        raw = f.read(8 * count)
        if len(raw) != 8 * count:
            raise ValueError("load_problem: truncated stream")
        return raw
    if tag in (2, 3):
        kappa, theta, zeta, xi = struct.unpack("<dddd", f.read(32))
        a = _sym_upper(take(n * n), n)
        g = np.frombuffer(take(n * p), dtype="<f8").reshape((n, p), order="F").copy(order="F")
        model = pcal.QuadraticModel(a, p, s, g0=None if tag == 3 else g)
        return model, {"tag": tag, "kappa": kappa, "theta": theta, "zeta": zeta, "xi": xi}
    if tag == 4:
        a = _sym_upper(take(n * n), n)
        b = _sym_upper(take(p * p), p)
        return pcal.BilinearModel(a, b, s), {"tag": tag}
    if tag in (1, 6):
        coeff, mode = struct.unpack("<dI", f.read(12))
        lmat = _sym_upper(take(n * n), n)
        model = pcal.DensityModel(lmat, p, coeff, s, variant="p6" if tag == 6 else "p1",
                                  mode="block-tridiag" if mode == 1 else "random-sym")
        return model, {"tag": tag, "coeff": coeff, "mode": mode}
    raise ValueError(f"load_problem: unknown kind tag {tag}")

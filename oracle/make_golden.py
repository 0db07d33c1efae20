"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    python -m oracle.make_golden            # small fixtures (seconds)
    python -m oracle.make_golden --cfg2     # + config-2 prefix (several minutes)

The fixtures pin the C restatement (tests/test_oracle_golden.py, CPU) and are
the parity anchors of the GPU tests.  Large matrices are stored as SHA-256 of
their little-endian bytes plus small slices.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

from oracle.oracle import Config, Model, Reference, MODEL_DENSE, MODEL_STENCIL, MODEL_KOHN_SHAM

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
TINY = np.finfo(float).tiny
INIT_SALT = 0x1235713      # harness.cpp:18
SPECTRAL_SALT = 0x73706563  # problems.cpp:19


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a, dtype="<f8").tobytes(order="F")).hexdigest()


def run_case(R: Reference, model: Model, x0, **cfg) -> dict:
    rep = R.solve(model, Config(**cfg), x0)
    out = {"trace": rep.trace[:, :6], "final_pre": rep.final_pre, "iterations": rep.iterations,
           "degenerate_steps": rep.degenerate_steps, "status": rep.status,
           "beta": rep.beta, "eta0": rep.eta0}
    out["final_post"] = rep.final_post if rep.final_post is not None else np.full(4, np.nan)
    if rep.final_x is not None:
        out["final_x_sha"] = sha(rep.final_x)
        out["stop_x_sha"] = sha(rep.stop_x)
    return out, rep


def small(R: Reference) -> None:
    os.makedirs(OUT, exist_ok=True)
    g = {}
    # --- RNG stream (rng.hpp, kernels.cpp:49-78)
    g["normal_seed1"] = R.random_normal(1001, 1, 1)[:, 0]
    g["normal_seed_init1"] = R.random_normal(21, 1, 1 ^ INIT_SALT)[:, 0]
    # --- kernels (kernels.cpp)
    a = R.random_normal(37, 5, 3)
    b = R.random_normal(37, 4, 4)
    g["k_a"], g["k_b"] = a, b
    g["k_matmul_at_b"] = R.matmul_at_b(a, b)
    g["k_gram"] = R.gram(a)
    c = R.random_normal(5, 6, 5)
    g["k_c"] = c
    g["k_matmul"] = R.matmul(a, c)
    x = R.random_normal(30, 4, 6)
    g["k_orth_x"] = x
    g["k_orth_q"] = R.orthonormalize(x)
    s50 = R.random_normal(50, 50, 7)
    sym = 0.5 * (s50 + s50.T)
    g["k_spec_a"] = np.asfortranarray(sym)
    g["k_spec_s"] = R.spectral_norm_estimate(sym, 11)
    # --- pcal_step known answers (test_solver.cpp:244-272 shapes)
    xs = R.random_normal(30, 5, 15)
    gs = R.random_normal(30, 5, 16)
    g["ps_x"], g["ps_g"] = xs, gs
    g["ps_out"], _ = R.pcal_step(xs, gs, 2.0)
    # --- stepsize_select closed forms (test_solver.cpp:167-224)
    X = np.array([[1.0], [1.0]]); Xp = np.zeros((2, 1)); G = np.array([[1.0], [3.0]]); Gp = np.zeros((2, 1))
    etas = []
    for kind, it in [(2, 1), (3, 1), (4, 1), (4, 2), (1, 2)]:
        etas.append(R.stepsize_select(Config(eta_kind=kind), it, 0.5, 0.25, X, Xp, G, Gp))
    g["ss_etas"] = np.array(etas)
    # --- cfg1 (n=1000, p=20, seed 1): the north-star CPU-runnable config
    m1 = R.dense_trace_min(1000, 20, 1)
    x01 = R.initial_point_qr(1000, 20, 1 ^ INIT_SALT)
    g["cfg1_s"] = m1.s
    g["cfg1_a_sha"] = sha(m1.a)
    g["cfg1_x0_sha"] = sha(x01)
    case, rep = run_case(R, m1, x01, tol_rel_kkt=TINY, max_iter=200, threads=8)
    for k, v in case.items():
        g["cfg1_" + k] = v
    g["cfg1_final_x_rows"] = rep.final_x[:8]
    g["cfg1_stop_x_rows"] = rep.stop_x[:8]
    # --- small dense cases from the reference's own tests
    cases = [("c40", 40, 5, 24, 25, {}), ("c12", 12, 2, 57, 58, {}),
             ("c20", 20, 4, 22, 23, {"max_iter": 40, "final_orth": False}),
             ("c14plam", 14, 3, 59, 60, {"multiplier_rule": 0}),
             ("c200", 200, 10, 101, 102, {})]
    for name, n, p, sa, sx, kw in cases:
        r = R.random_normal(n, n, sa)
        A = np.asfortranarray(0.5 * (r + r.T))
        s = R.spectral_norm_estimate(A, SPECTRAL_SALT)  # make_quadratic default (problems.cpp:292)
        mod = Model(MODEL_DENSE, n, p, s, a=A)
        x0 = R.initial_point_qr(n, p, sx)
        cfg = {"threads": 1}
        cfg.update(kw)
        case, rep = run_case(R, mod, x0, **cfg)
        g[name + "_a_seed"] = sa
        g[name + "_x0_seed"] = sx
        g[name + "_s"] = s
        for k, v in case.items():
            g[name + "_" + k] = v
        if rep.final_x is not None:
            g[name + "_final_x"] = rep.final_x
            g[name + "_stop_x"] = rep.stop_x
    # stationary start: A = Diag(1,2,3,4), X = [e1 e2] (test_solver.cpp:318-331)
    A4 = np.diag([1.0, 2.0, 3.0, 4.0])
    X4 = np.zeros((4, 2)); X4[0, 0] = 1.0; X4[1, 1] = 1.0
    case, _ = run_case(R, Model(MODEL_DENSE, 4, 2, 4.0, a=np.asfortranarray(A4)), X4)
    for k, v in case.items():
        g["stat_" + k] = v
    np.savez_compressed(os.path.join(OUT, "reference_small.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_small.npz"), len(g), "arrays")


def algorithm_cases(R: Reference) -> None:
    """PLAM, PLAM-DA, PCAL-DA, MOptQR and PCAL with the PLAM multiplier formula
    (solver.cpp:320-474) on the config-1 instance and a small converging case."""
    from oracle.oracle import ALG_PLAM, ALG_PCAL, ALG_MOPTQR, ALG_PLAMDA, ALG_PCALDA
    g = {}
    m1 = R.dense_trace_min(1000, 20, 1, s=44.26282919872377)
    x01 = R.initial_point_qr(1000, 20, 1 ^ INIT_SALT)
    r = R.random_normal(40, 40, 24)
    a40 = np.asfortranarray(0.5 * (r + r.T))
    s40 = R.spectral_norm_estimate(a40, SPECTRAL_SALT)
    m40 = Model(MODEL_DENSE, 40, 5, s40, a=a40)
    x040 = R.initial_point_qr(40, 5, 25)
    algs = {"plam": (ALG_PLAM, 1), "plamda": (ALG_PLAMDA, 1), "pcalda": (ALG_PCALDA, 1),
            "moptqr": (ALG_MOPTQR, 1), "pcalplamf": (ALG_PCAL, 0)}
    for name, (alg, mult) in algs.items():
        case, rep = run_case(R, m1, x01, tol_rel_kkt=TINY, max_iter=60, threads=8, algorithm=alg,
                             multiplier_rule=mult)
        for k, v in case.items():
            g[f"a1_{name}_{k}"] = v
        case, rep = run_case(R, m40, x040, algorithm=alg, multiplier_rule=mult, max_iter=3000)
        for k, v in case.items():
            g[f"a40_{name}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "reference_algorithms.npz"), **g)
    print("wrote reference_algorithms.npz")


ALM_CASES = {  # name: (instance, AlmOptions(inner_max, outer_max, scale), config overrides)
    "a40_default": ("a40", (500, 50, 0.1), {}),
    "a40_tight_caps": ("a40", (6, 5, 0.1), {}),                 # inner caps, outer cap ⇒ MaxIter
    "a40_budget": ("a40", (500, 50, 0.01), {"max_iter": 25}),  # iteration budget inside a loop
    "a40_beta0": ("a40", (500, 50, 0.1), {"beta": 0.0, "max_iter": 300}),
    "c1_caps": ("c1", (7, 50, 0.1), {"max_iter": 60, "threads": 8}),
}


def alm_cases(R: Reference) -> None:
    """ALM (alm_outer, solver.cpp:478-624) through the reference's solve(): traces,
    finals, the outer / cap counters — including the reference unit tests'
    instances (test_solver.cpp:463-498)."""
    import ctypes as C
    from oracle.oracle import ALG_ALM
    L = R.lib
    L.ref_set_alm.argtypes = [C.c_int, C.c_int, C.c_double]
    L.ref_last_alm_counts.argtypes = [C.POINTER(C.c_int64)]
    r = R.random_normal(40, 40, 24)
    a40 = np.asfortranarray(0.5 * (r + r.T))
    s40 = R.spectral_norm_estimate(a40, SPECTRAL_SALT)
    inst = {"a40": (Model(MODEL_DENSE, 40, 5, s40, a=a40), R.initial_point_qr(40, 5, 25)),
            "c1": (R.dense_trace_min(1000, 20, 1, s=44.26282919872377),
                   R.initial_point_qr(1000, 20, 1 ^ INIT_SALT))}
    g = {}
    for name, (which, (imax, omax, scale), over) in ALM_CASES.items():
        model, x0 = inst[which]
        L.ref_set_alm(imax, omax, scale)
        case, rep = run_case(R, model, x0, algorithm=ALG_ALM, **over)
        cnt = (C.c_int64 * 2)()
        L.ref_last_alm_counts(cnt)
        for k, v in case.items():
            g[f"{name}_{k}"] = v
        g[f"{name}_counts"] = np.array([cnt[0], cnt[1]])
    L.ref_set_alm(500, 50, 0.1)
    np.savez_compressed(os.path.join(OUT, "reference_alm.npz"), **g)
    print("wrote reference_alm.npz")


def container_cases(R: Reference) -> None:
    """OCPROB01 containers of the Bilinear / Density models (problems.cpp:341-416)."""
    import ctypes as C
    L = R.lib
    L.ref_save_generated.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                     C.c_uint64, C.c_char_p]
    for name, args in {"p4": (4, 12, 3, 1.0, 0, 41), "p1": (1, 10, 2, 1.5, 1, 42),
                       "p6": (6, 11, 3, 1.0, 0, 43)}.items():
        path = os.path.join(OUT, f"ref_{name}.ocprob")
        assert L.ref_save_generated(*args, path.encode()) == 0, name
    print("wrote ref_p4/p1/p6.ocprob")


def matrix_case(R: Reference) -> None:
    """run_matrix (harness.cpp:75-104) summary CSV of a small fixed matrix."""
    import ctypes as C
    L = R.lib
    L.ref_run_matrix_csv.argtypes = [C.c_char_p, C.c_int64]
    buf = C.create_string_buffer(1 << 20)
    assert L.ref_run_matrix_csv(buf, len(buf)) == 0
    open(os.path.join(OUT, "ref_matrix.csv"), "w").write(buf.value.decode())
    print("wrote ref_matrix.csv")


def report_io_cases(R: Reference) -> None:
    """The reference's JSON / CSV report text and an OCPROB01 container."""
    import ctypes as C
    L = R.lib
    L.ref_run_single_text.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int64, C.c_char_p,
                                      C.c_int64, C.c_char_p, C.c_int64]
    L.ref_save_quadratic.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double,
                                     C.c_char_p]
    jb, cb = C.create_string_buffer(1 << 20), C.create_string_buffer(1 << 20)
    assert L.ref_run_single_text(60, 4, 7, 50, jb, len(jb), cb, len(cb)) == 0
    open(os.path.join(OUT, "ref_report_p1_n60.json"), "w").write(jb.value.decode() + "\n")
    open(os.path.join(OUT, "ref_trace_p1_n60.csv"), "w").write(cb.value.decode())
    r = R.random_normal(40, 40, 31)
    a = np.asfortranarray(0.5 * (r + r.T))
    g0 = R.random_normal(40, 5, 32)
    s = R.spectral_norm_estimate(a, 33)
    path = os.path.join(OUT, "ref_quad40.ocprob")
    assert L.ref_save_quadratic(a.ctypes.data, g0.ctypes.data, 40, 5, s, path.encode()) == 0
    np.savez_compressed(os.path.join(OUT, "ref_quad40.npz"), a=a, g0=g0, s=s)
    print("wrote report/container fixtures")


JSON_MAGNITUDES = [1e15, 1.5e15, 9.999e15, 1e16, 1e14, 999999999999999.9, 1234567890123456.0,
                   -2.5e15, 123456.789, 1e-4, 1e-5, 1.5e-5, 0.1, 100.0, 1e300, 5e-324, -0.0,
                   0.0, 1e21, 4.7429826849363259e-05, -418.65544567286281]


def json_magnitudes_case(R: Reference) -> None:
    """The reference's to_json number formatting over magnitudes where Python's
    repr and nlohmann's dtoa disagree (1e15 ≤ |v| < 1e16) and their neighbours."""
    import ctypes as C
    L = R.lib
    L.ref_report_json_values.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_int64]
    v = np.array(JSON_MAGNITUDES)
    jb = C.create_string_buffer(1 << 20)
    assert L.ref_report_json_values(v.ctypes.data, len(v), jb, len(jb)) == 0
    open(os.path.join(OUT, "ref_report_magnitudes.json"), "w").write(jb.value.decode() + "\n")
    print("wrote ref_report_magnitudes.json")


def init_cases(R: Reference) -> None:
    """initial_point(InitialPointSpec) for the three InitMode values (solver.cpp:136-170)."""
    import ctypes as C
    g = {}
    for name, mode, sigma, n, p, seed in [("qr", 0, 0.5, 30, 4, 11), ("a2i", 1, 0.6, 30, 4, 12),
                                          ("a2ii", 2, 0.5, 31, 5, 13), ("a2ii_p1", 2, 0.5, 8, 1, 14)]:
        out = np.zeros((n, p), order="F")
        assert R.lib.ref_initial_point(mode, sigma, seed, n, p,
                                       out.ctypes.data_as(C.POINTER(C.c_double))) == 0
        g[name] = out
        g[name + "_args"] = np.array([mode, sigma, n, p, seed], dtype=float)
    np.savez_compressed(os.path.join(OUT, "reference_init.npz"), **g)
    print("wrote reference_init.npz")


HARNESS_CASES = {  # name: (kind, n, p, alpha, kappa, theta, zeta, xi, block_tridiag, seed, init, sigma, iters)
    "p1_alpha0": (1, 80, 5, 0.0, 1.0, 1.01, 1.01, 1.0, 0, 11, 0, 0.5, 60),
    "p1_block": (1, 60, 4, 0.0, 1.0, 1.01, 1.01, 1.0, 1, 12, 0, 0.5, 3000),
    "p2": (2, 90, 6, 0.0, 2.0, 1.05, 1.02, 0.7, 0, 13, 0, 0.5, 3000),
    "p3_a2i": (3, 70, 4, 0.0, 0.0, 1.08, 1.0, 0.5, 0, 14, 1, 0.6, 3000),
    # DensityModel (P1 α > 0: LU path; block operator: Cholesky path) and P6, BilinearModel P4
    "p1_alpha1": (1, 80, 5, 1.0, 1.0, 1.01, 1.01, 1.0, 0, 21, 0, 0.5, 3000),
    "p1_block_alpha2": (1, 60, 4, 2.0, 1.0, 1.01, 1.01, 1.0, 1, 22, 0, 0.5, 3000),
    "p4": (4, 60, 5, 1.0, 1.0, 1.01, 1.01, 1.0, 0, 23, 0, 0.5, 3000),
    "p6": (6, 70, 4, 1.0, 1.0, 1.01, 1.01, 1.0, 0, 24, 0, 0.5, 3000),
    "p6_block_a2ii": (6, 50, 3, 1.0, 1.0, 1.01, 1.01, 1.0, 1, 25, 2, 0.5, 3000),
}


def harness_cases(R: Reference) -> None:
    """run_single (harness.cpp:62-73) JSON reports for every problem kind."""
    import ctypes as C
    L = R.lib
    L.ref_run_single_json.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_int, C.c_uint64,
                                      C.c_int, C.c_double, C.c_int64, C.c_char_p, C.c_int64]
    for name, (kind, n, p, alpha, kappa, theta, zeta, xi, bt, seed, init, sigma, iters) in \
            HARNESS_CASES.items():
        buf = C.create_string_buffer(1 << 22)
        assert L.ref_run_single_json(kind, n, p, alpha, kappa, theta, zeta, xi, bt, seed, init,
                                     sigma, iters, buf, len(buf)) == 0, name
        open(os.path.join(OUT, f"ref_run_single_{name}.json"), "w").write(buf.value.decode() + "\n")
    print("wrote run_single reports")


def harness_ensembles(R: Reference, k: int = 8) -> None:
    """For every run_single case: the iteration count and post-orth objective of
    the reference solve() from the run_single start point and from K copies of
    it with one entry moved by one ulp — how far a converging run's step count
    moves under rounding-level differences (the GPU's tolerance)."""
    import ctypes as C
    from types import SimpleNamespace
    L = R.lib
    L.ref_make_problem.restype = C.c_void_p
    L.ref_make_problem.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_double, C.c_int, C.c_uint64]
    g = {}
    for name, (kind, n, p, alpha, kappa, theta, zeta, xi, bt, seed, init, sigma, iters) in \
            HARNESS_CASES.items():
        h = L.ref_make_problem(kind, n, p, alpha, kappa, theta, zeta, xi, bt, seed)
        assert h, name
        x0 = np.empty((n, p), order="F")
        assert L.ref_initial_point(init, sigma, seed ^ INIT_SALT, n, p,
                                   x0.ctypes.data_as(C.POINTER(C.c_double))) == 0
        its, fpost = [], []
        for q in range(k + 1):
            xp = x0.copy(order="F")
            if q > 0:
                e = (q * 2654435761) % xp.size
                xp.flat[e] = np.nextafter(xp.flat[e], np.inf if q % 2 else -np.inf)
            cfg = Config(max_iter=iters, threads=1)
            rep, keep = R._report(SimpleNamespace(n=n, p=p), cfg, ())
            assert L.ref_solve(C.c_void_p(h), C.byref(cfg.c()), xp.ctypes.data_as(C.POINTER(C.c_double)),
                               C.byref(rep), None) == 0, name
            out = R._finish(rep, keep, ())
            its.append(out.iterations)
            fpost.append(out.final_post[0] if out.final_post is not None else np.nan)
        L.ref_free_model(C.c_void_p(h))
        g[name + "_iterations"] = np.array(its)
        g[name + "_final_post_f"] = np.array(fpost)
        print(name, its)
    np.savez_compressed(os.path.join(OUT, "reference_run_single_ensembles.npz"), **g)
    print("wrote reference_run_single_ensembles.npz")


def linsolve_cases(R: Reference) -> None:
    """LinearSolver (linsolve.cpp) inverses: random symmetric (LU path), the block
    operator (Cholesky path), a singular matrix (generation_error)."""
    import ctypes as C
    L = R.lib
    dp = C.POINTER(C.c_double)
    L.ref_linear_inverse.argtypes = [dp, C.c_int64, dp]
    from oracle.oracle import Restatement
    O = Restatement()
    g = {}
    blk = np.zeros((30, 30), order="F")
    for b in range(0, 30, 5):
        for i in range(5):
            blk[b + i, b + i] = 2.0
            if i < 4:
                blk[b + i, b + i + 1] = blk[b + i + 1, b + i] = -1.0
    sing = np.ones((6, 6), order="F")
    m = O.random_normal(40, 40, 5)
    for name, a in [("lu", 0.5 * (m + m.T)),
                    ("chol", blk), ("singular", sing)]:
        a = np.asfortranarray(a)
        out = np.zeros_like(a, order="F")
        rc = L.ref_linear_inverse(a.ctypes.data_as(dp), a.shape[0], out.ctypes.data_as(dp))
        g[name + "_a"] = a
        g[name + "_inv"] = out
        g[name + "_singular"] = np.array(rc == 1)
    np.savez_compressed(os.path.join(OUT, "reference_linsolve.npz"), **g)
    print("wrote reference_linsolve.npz")


MODEL_EVAL_CASES = {  # name: (kind, n, p, alpha, block_tridiag, seed) — acceptance #3's instances
    "p1": (1, 60, 6, 1.0, 0, 31), "p6": (6, 60, 6, 1.0, 0, 32), "p4": (4, 60, 6, 1.0, 0, 35),
    "p1_block": (1, 45, 4, 2.0, 1, 36), "p6_block": (6, 45, 4, 1.0, 1, 37),
}


def model_eval_cases(R: Reference) -> None:
    """The reference's P1 (α > 0) / P4 / P6 models evaluated at seeded points."""
    import ctypes as C
    L = R.lib
    dp = C.POINTER(C.c_double)
    L.ref_evaluate_problem.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                       C.c_uint64, dp, dp, dp, dp]
    g = {}
    for name, (kind, n, p, alpha, bt, seed) in MODEL_EVAL_CASES.items():
        x = np.asfortranarray(R.random_normal(n, p, 300 + seed))
        f, fd = C.c_double(), C.c_double()
        gr = np.zeros((n, p), order="F")
        assert L.ref_evaluate_problem(kind, n, p, alpha, bt, seed, x.ctypes.data_as(dp),
                                      C.byref(f), gr.ctypes.data_as(dp), C.byref(fd)) == 0, name
        g[name + "_x"] = x
        g[name + "_f"] = f.value
        g[name + "_g"] = gr
        g[name + "_fd"] = fd.value  # fd_gradient_check(model, x) with the reference defaults
    np.savez_compressed(os.path.join(OUT, "reference_models.npz"), **g)
    print("wrote reference_models.npz")


DIAG_CASES = {  # name: (kind, n, p, alpha, block, seed, x-kind, beta)
    "p1_near": (1, 60, 6, 1.0, 0, 31, "near", 30.0),   # near-orthonormal x: the bound applies
    "p4_far": (4, 60, 6, 1.0, 0, 35, "randn", 1.0),    # random x: not applicable
    "p6_near": (6, 45, 4, 1.0, 1, 37, "near", 20.0),
}


def diagnostics_cases(R: Reference) -> None:
    """kkt_violation, feasibility_violation, merit_h, feasibility_bound_check
    (diagnostics.cpp:21-98) of the reference's models at seeded points."""
    import ctypes as C
    L = R.lib
    dp = C.POINTER(C.c_double)
    L.ref_diagnostics.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_int, C.c_uint64,
                                  dp, C.c_double, dp]
    g = {}
    for name, (kind, n, p, alpha, bt, seed, xk, beta) in DIAG_CASES.items():
        if xk == "near":  # orthonormal start plus a small perturbation
            x = R.initial_point_qr(n, p, seed + 100) + 1e-3 * R.random_normal(n, p, seed + 200)
        else:
            x = R.random_normal(n, p, seed + 300)
        x = np.asfortranarray(x)
        out = np.zeros(9)
        assert L.ref_diagnostics(kind, n, p, alpha, bt, seed, x.ctypes.data_as(dp), beta,
                                 out.ctypes.data_as(dp)) == 0, name
        g[name + "_x"] = x
        g[name + "_out"] = out
    np.savez_compressed(os.path.join(OUT, "reference_diagnostics.npz"), **g)
    print("wrote reference_diagnostics.npz")


def grid_cases(R: Reference) -> None:
    """Grid models (no reference implementation): the reference solve() driving
    the restated operator — pins the PCAL loop around it, not the operator."""
    g = {}
    for name, kind, grid, p in [("st6", MODEL_STENCIL, (6, 5, 4), 4),
                                ("ks6", MODEL_KOHN_SHAM, (6, 6, 6), 4)]:
        n = grid[0] * grid[1] * grid[2]
        from oracle.oracle import Restatement
        O = Restatement()
        v = O.random_uniform(n, 3) if kind == MODEL_STENCIL else -O.random_uniform(n, 3)
        s = 12.0 + float(np.max(np.abs(v)))
        mod = Model(kind, n, p, s, grid=grid, v=v)
        x0 = R.initial_point_qr(n, p, 3 ^ INIT_SALT)
        case, rep = run_case(R, mod, x0, tol_rel_kkt=TINY, max_iter=60)
        g[name + "_v"] = v
        g[name + "_s"] = s
        for k, val in case.items():
            g[name + "_" + k] = val
        g[name + "_final_x"] = rep.final_x
    np.savez_compressed(os.path.join(OUT, "reference_grid.npz"), **g)
    print("wrote reference_grid.npz")


def cfg2(R: Reference) -> None:
    """Config 2 (n=16384, p=128, seed 1): s and the first iterations."""
    import time
    t = time.time()
    m = R.dense_trace_min(16384, 128, 1, threads=16)
    print("cfg2 gen + s:", time.time() - t, m.s, flush=True)
    x0 = R.initial_point_qr(16384, 128, 1 ^ INIT_SALT)
    t = time.time()
    case, rep = run_case(R, m, x0, tol_rel_kkt=TINY, max_iter=3, threads=16, final_orth=False)
    print("cfg2 3 iters:", time.time() - t, flush=True)
    g = {"cfg2_s": m.s, "cfg2_a_sha": sha(m.a), "cfg2_x0_sha": sha(x0)}
    for k, v in case.items():
        g["cfg2_" + k] = v
    g["cfg2_stop_x_rows"] = rep.stop_x[:8]
    np.savez_compressed(os.path.join(OUT, "reference_cfg2.npz"), **g)
    print("wrote reference_cfg2.npz")


def grids_full(R: Reference) -> None:
    """Configs 3 and 4 at full size (64³×256 stencil, 48³×512 Kohn–Sham):
    the reference solve() driving the restated operators for 3 iterations.  The
    instances are the product's definitions (paper_1810_03930_b200/problems.py)
    built from the reference's random stream."""
    import time
    from oracle.oracle import Restatement
    from paper_1810_03930_b200.problems import ks_potential
    O = Restatement()
    g = {}
    for name, kind, grid, p in [("cfg3", MODEL_STENCIL, (64, 64, 64), 256),
                                ("cfg4", MODEL_KOHN_SHAM, (48, 48, 48), 512)]:
        n = grid[0] * grid[1] * grid[2]
        if kind == MODEL_STENCIL:
            v = O.random_uniform(n, 1)
            s = 12.0 + float(np.max(v))
        else:
            v = ks_potential(grid, 1, O)
            s = 6.0 + float(np.max(np.abs(v)))
        t = time.time()
        x0 = O.initial_point_qr(n, p, 1 ^ INIT_SALT, threads=16)
        print(name, "x0:", time.time() - t, flush=True)
        t = time.time()
        case, rep = run_case(R, Model(kind, n, p, s, grid=grid, v=v), x0, tol_rel_kkt=TINY,
                             max_iter=3, threads=16, final_orth=False)
        print(name, "3 iters:", time.time() - t, flush=True)
        g[name + "_v_sha"] = sha(v)
        g[name + "_x0_sha"] = sha(x0)
        g[name + "_s"] = s
        for k, val in case.items():
            g[name + "_" + k] = val
        g[name + "_stop_x_rows"] = rep.stop_x[:8]
    np.savez_compressed(os.path.join(OUT, "reference_grids_full.npz"), **g)
    print("wrote reference_grids_full.npz")


if __name__ == "__main__":
    R = Reference()
    small(R)
    grid_cases(R)
    algorithm_cases(R)
    report_io_cases(R)
    json_magnitudes_case(R)
    init_cases(R)
    harness_cases(R)
    harness_ensembles(R)
    linsolve_cases(R)
    model_eval_cases(R)
    alm_cases(R)
    matrix_case(R)
    diagnostics_cases(R)
    container_cases(R)
    if "--cfg2" in sys.argv:
        cfg2(R)
    if "--grids" in sys.argv:
        grids_full(R)

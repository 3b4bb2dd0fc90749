"""Generates the golden fixtures under tests/golden/ from the reference itself.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_golden.py

Every number comes from the reference's own code compiled in place
(oracle/_ref/libirkref.so, oracle/Makefile): Butcher tables and coefficient
matrices (butcher.cpp), assembled M/K (fem.cpp), AMG hierarchies (amg.cpp) and
IRK steps (irk.cpp + gmres.cpp behind the GMRES(m) restart harness).  Matrices
and hierarchies are stored as SHA-256 digests of their raw arrays (bit-exact
pins without committing megabytes); step results are stored in full.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from refs import Ref, RefSolver  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def heat_u0(n_cells: int, noise: float, seed: int) -> np.ndarray:
    # the project-defined u0 (paper_2010_11377_b200.ProblemSetup.initial)
    import paper_2010_11377_b200 as P
    return P.make_heat_setup(n_cells).initial(noise, seed)


def main():
    out = {}
    # Butcher tables and coefficients (butcher.cpp:29-101, 190-288)
    for scheme, ss in ((0, range(1, 8)), (1, range(2, 6))):
        for s in ss:
            A, b, c, q = Ref.tableau(scheme, s)
            out[f"tab_{scheme}_{s}_A"], out[f"tab_{scheme}_{s}_b"], out[f"tab_{scheme}_{s}_c"] = A, b, c
            for kind in range(4):
                At, st = Ref.precond_coeff(scheme, s, kind)
                out[f"coeff_{scheme}_{s}_{kind}"] = At
                out[f"struct_{scheme}_{s}_{kind}"] = np.array(st)
    np.savez_compressed(HERE / "butcher.npz", **out)

    # Problems, hierarchies and steps
    cases = [
        # name, kind, cells, scheme, s, coeff kind, ht, noise, seed, restart
        ("c1_heat64_radau2_ld", "heat", 64, 0, 2, 3, 0.01, 0.0, 1, 50),
        ("heat48_radau3_gsl_noise", "heat", 48, 0, 3, 1, 0.005, 0.01, 3, 50),
        ("heat48_radau3_ld_restart5", "heat", 48, 0, 3, 3, 0.01, 0.01, 9, 5),
        ("heat48_lobatto4_du", "heat", 48, 1, 4, 2, 0.005, 0.01, 3, 50),
        ("heat48_radau3_jacobi", "heat", 48, 0, 3, 0, 0.005, 0.01, 3, 50),
        ("dg64_radau2_ld", "dg", 64, 0, 2, 3, 0.01, 0.0, 1, 50),
    ]
    # extras: side (GMRES preconditioning side) and a time-dependent forcing
    # cos(t) * fq at t_n (ref_harness.cpp cos_forcing)
    extras = {
        "heat48_radau3_ld_left": dict(side="left"),
        "heat48_radau3_ld_left_restart5": dict(side="left"),
        "heat32_radau3_ld_forced": dict(t_n=0.37, fq_seed=11),
    }
    cases += [
        ("heat48_radau3_ld_left", "heat", 48, 0, 3, 3, 0.01, 0.01, 5, 50),
        ("heat48_radau3_ld_left_restart5", "heat", 48, 0, 3, 3, 0.01, 0.01, 5, 5),
        ("heat32_radau3_ld_forced", "heat", 32, 0, 3, 3, 0.01, 0.01, 2, 50),
    ]
    for name, kind, cells, scheme, s, ck, ht, noise, seed, restart in cases:
        prob = Ref.problem(kind, cells, 0.005)
        g = {"cells": np.array(cells), "scheme": np.array(scheme), "s": np.array(s),
             "kind": np.array(ck), "ht": np.array(ht), "restart": np.array(restart)}
        g["M_sha"] = np.array(digest(*prob["M"]))
        g["K_sha"] = np.array(digest(*prob["K"]))
        g["f_lift_sha"] = np.array(digest(prob["f_lift"]))
        # hierarchy of each distinct diagonal block M + ht*d*K (stage.cpp:85-106)
        At, _ = Ref.precond_coeff(scheme, s, ck)
        distinct = []
        for j in range(s):
            if At[j, j] not in distinct:
                distinct.append(At[j, j])
        for k, d in enumerate(distinct):
            rp, ci, mv = prob["M"]
            B = (rp, ci, 1.0 * mv + (ht * d) * prob["K"][2])
            h = Ref.amg(B)
            sizes, shas = [], []
            for l in range(h.n_levels()):
                (a, _), = [h.level(l, "A")]
                sizes.append(len(a[0]) - 1)
                parts = [*a, h.inv_diag(l)]
                if l + 1 < h.n_levels():
                    parts += [*h.level(l, "P")[0], *h.level(l, "R")[0]]
                shas.append(digest(*parts))
            g[f"hier{k}_sizes"] = np.array(sizes)
            g[f"hier{k}_sha"] = np.array(shas)
        u0 = np.zeros(len(prob["M"][0]) - 1) if kind == "dg" else heat_u0(cells, noise, seed)
        rs = RefSolver(prob["M"], prob["K"], scheme, s, ck, ht)
        ex = extras.get(name, {})
        side = ex.get("side", "right")
        t_n = ex.get("t_n", 0.0)
        fq = (np.random.default_rng(ex["fq_seed"]).uniform(-1.0, 1.0, len(u0))
              if "fq_seed" in ex else None)
        r = rs.step(u0, prob["f_lift"], restart=restart, side=side, t_n=t_n, fq=fq)
        g.update(u0=u0, u_next=r["u_next"], K=r["K"], iterations=np.array(r["iterations"]),
                 cycles=np.array(r["cycles"]), true_rel=np.array(r["true_rel"]),
                 history=r["history"], side=np.array(side), t_n=np.array(t_n))
        if fq is not None:
            g["fq"] = fq
        np.savez_compressed(HERE / f"{name}.npz", **g)
        print(name, "iterations", r["iterations"], "cycles", r["cycles"], "levels",
              [g[f"hier{k}_sizes"].tolist() for k in range(len(distinct))])


def trajectory():
    """The reference's own integrate (irk.cpp:70-102) with a truncated last
    step and the cos(t) * fq forcing: heat 24^2, Radau IIA s=2, P_LD,
    h_t = 0.01, t_final = 0.035 (steps 0.01, 0.01, 0.01, ~0.005)."""
    cells, s, ht, t_final = 24, 2, 0.01, 0.035
    prob = Ref.problem("heat", cells)
    u0 = heat_u0(cells, 0.01, 4)
    fq = np.random.default_rng(5).uniform(-1.0, 1.0, len(u0))
    t, steps = 0.0, []
    while t < t_final - 1e-14 * t_final:
        st = ht if t + ht <= t_final else t_final - t
        steps.append(st)
        t += st
    main_s = RefSolver(prob["M"], prob["K"], 0, s, 3, ht)
    trunc = RefSolver(prob["M"], prob["K"], 0, s, 3, steps[-1])
    r = main_s.integrate(u0, t_final, trunc=trunc, lift=prob["f_lift"], fq=fq)
    np.savez_compressed(HERE / "traj_heat24_radau2_ld_forced.npz", cells=np.array(cells),
                        s=np.array(s), ht=np.array(ht), t_final=np.array(t_final), u0=u0, fq=fq,
                        u_final=r["u_final"], steps=np.array(r["steps"]),
                        t_end=np.array(r["t_final"]), iterations=np.array(r["iterations"]))
    print("trajectory steps", r["steps"], "iterations", r["iterations"])


if __name__ == "__main__":
    main()
    trajectory()

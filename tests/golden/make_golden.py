"""Regenerate the committed golden fixtures (run in the build container, where the reference
tree exists):  python tests/golden/make_golden.py

* spec_kats.json -- the known-answer examples of the reference's behavioural spec
  (/root/reference/SPEC.md; line numbers below), written out as numbers.  These are the
  only known answers the reference ships for the hot path.
* wave_bands_ref.npz -- cubic/quadratic spline Gram bands produced by the REFERENCE'S OWN
  stk/splines.hpp + stk/quadrature.hpp compiled as oracle/_ref/libstkref.so (the spline_gram
  loop of stk/discretize.hpp:111-131 restated around them), incl. the config-4 size.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402


def spec_kats():
    return {
        "heat_time_matrices": [
            {"src": "SPEC.md:129", "nt": 1, "T": 1.0, "D": [[1.0]], "C": [[0.5]]},
            {"src": "SPEC.md:130", "nt": 3, "T": 3.0,
             "D": [[1, -1, 0], [0, 1, -1], [0, 0, 1]],
             "C": [[0.5, 0.5, 0], [0, 0.5, 0.5], [0, 0, 0.5]]},
            {"src": "SPEC.md:131", "nt": 6, "T": 1.0, "D_row_sums": [0, 0, 0, 0, 0, 1]},
        ],
        "fem1d_matrices": [
            {"src": "SPEC.md:138", "a": 0.0, "b": 1.0, "nh": 1, "A": [[4.0]], "M": [[1.0 / 3.0]]},
            {"src": "SPEC.md:139", "a": 0.0, "b": 1.0, "nh": 3,
             "A": [[8, -4, 0], [-4, 8, -4], [0, -4, 8]]},
            {"src": "SPEC.md:140", "a": 0.0, "b": 1.0, "nh": 7, "M_interior_row_sum": 0.125},
        ],
        "solve_projected_heat": [
            {"src": "SPEC.md:307", "H_M": [[1.0]], "H_A": [[1.0]], "D": [[1.0]], "C": [[1.0]],
             "G": [[2.0]], "Y": [[1.0]]},
            {"src": "SPEC.md:308", "H_M": [[1, 0], [0, 1]], "H_A": [[1, 0], [0, 2]], "nt": 3,
             "T": 3.0, "G": "ones", "oracle": "dense Kronecker solve"},
            {"src": "SPEC.md:309", "k": 5, "nt": 7, "residual_max": 1e-11},
        ],
        "two_term_solve": [
            {"src": "SPEC.md:325", "M_h": [[1.0]], "Q_h": [[1.0]], "M_t": [[1.0]], "Q_t": [[1.0]],
             "V": [[2.0]], "W": [[1.0]]},
            {"src": "SPEC.md:326", "identity": True, "W_over_V": 0.5},
            {"src": "SPEC.md:327", "nh": 6, "nt": 4, "tol": 1e-9},
        ],
        "apply_kron": [{"src": "SPEC.md:298", "single_term_identity": True}],
        "wave_operator_apply": [{"src": "SPEC.md:462", "identity_like_gain": 2.0}],
        "gmres": [
            {"src": "SPEC.md:453", "apply": "identity", "iterations": 1},
            {"src": "SPEC.md:454", "apply": "diag(1..5)", "b": "ones", "max_iterations": 5,
             "tol": 1e-10},
        ],
        "crank_nicolson": [
            {"src": "SPEC.md:517", "M": 1.0, "A": 0.0, "nt": 8, "T": 1.0, "u": "l*dt"},
            {"src": "SPEC.md:518", "M": 1.0, "A": 1.0, "u0": 1.0, "u": "((1-dt/2)/(1+dt/2))^l"},
        ],
    }


def main():
    (HERE / "spec_kats.json").write_text(json.dumps(spec_kats(), indent=1) + "\n")
    out = {}
    for nh, nt, deg in [(16, 16, 3), (8, 5, 2), (31, 33, 3), (1023, 1024, 3)]:
        sb, tb = O.ref_wave_bands(nh, nt, deg)
        out[f"space_{nh}_{deg}"] = sb
        out[f"time_{nt}_{deg}"] = tb
    lib = O.ref_lib()
    import ctypes as C
    for npts in (3, 4, 6):  # 6: project_rhs_heat's default rule (stk/rhs_sep.hpp:113)
        x, w = np.zeros(npts), np.zeros(npts)
        lib.ref_gauss_legendre(npts, 0.0, 1.0, x.ctypes.data_as(C.POINTER(C.c_double)),
                               w.ctypes.data_as(C.POINTER(C.c_double)))
        out[f"gauss_{npts}_x"], out[f"gauss_{npts}_w"] = x, w
    np.savez_compressed(HERE / "wave_bands_ref.npz", **out)
    print("wrote", HERE / "spec_kats.json", HERE / "wave_bands_ref.npz")


if __name__ == "__main__":
    main()

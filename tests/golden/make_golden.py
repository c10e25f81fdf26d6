"""Regenerates the golden fixtures from the UNMODIFIED reference library
(oracle/_ref/libsdg_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run in the build container:  python tests/golden/make_golden.py

Fixtures (npz, small):
  ref2d_<name>.npz : 2D reference fields for z-invariant embedding checks —
                     initial state, residual at t_res, state after n_steps of dt.
  ref_mortar_ops.npz : build_mortar_operators for N=1..7 (LGL, Gauss), sigma set.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as P  # noqa: E402
from paper_2008_04356_b200 import types as T  # noqa: E402

BANDS3 = [(2, 1.0, 0.0), (2, 1.0, 1.0), (2, 1.0, 0.0)]

# name -> (bands, ny, degree, kind, mu, periodic_x, case, t_res, dt, n_steps)
CASES = {
    "dw_lgl3_inv": (BANDS3, 6, 3, T.NODES_LGL, 0.0, True, "density_wave", 0.37, 0.004, 10),
    "dw_gauss3_visc": (BANDS3, 6, 3, T.NODES_GAUSS, 1e-3, True, "density_wave", 0.37, 0.004, 10),
    "dw_gauss5_visc_dirichlet": ([(2, 1.0, 0.0), (2, 1.0, 0.5)], 2, 5, T.NODES_GAUSS, 1e-3, False, "density_wave",
                                 0.05, 0.002, 10),
    "fs_lgl4_inv": (BANDS3, 6, 4, T.NODES_LGL, 0.0, True, "freestream", 0.99, 0.006437725221731195, 20),
}


def main():
    for name, (bands, ny, deg, kind, mu, px, case, t_res, dt, n) in CASES.items():
        spec = P.ref_spec(bands, ny, deg, kind, mu=mu, periodic=(px, True), case=case)
        ref = P.Ref2D(spec)
        u0 = ref.initial(0.0)
        res = ref.residual(0.0, t_res)
        un, t_end, rebuilds = ref.steps(0.0, dt, n)
        np.savez_compressed(os.path.join(HERE, f"ref2d_{name}.npz"), u0=u0, residual=res, u_end=un, t_res=t_res,
                            dt=dt, n_steps=n, t_end=t_end, rebuilds=rebuilds)
    sig = np.array([-1.0, -0.75, -0.3, 0.0, 0.21, 0.37, 0.9, 0.999])
    ops = {}
    for kind in (T.NODES_LGL, T.NODES_GAUSS):
        for deg in range(1, 8):
            f = []
            b = []
            for s in sig:
                ff, bb = P.ref_mortar_ops(deg, kind, float(s))
                f.append(ff)
                b.append(bb)
            ops[f"fwd_{kind}_{deg}"] = np.array(f)
            ops[f"bwd_{kind}_{deg}"] = np.array(b)
    np.savez_compressed(os.path.join(HERE, "ref_mortar_ops.npz"), sigma=sig, **ops)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()

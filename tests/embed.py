"""z-invariant embedding of the reference's 2D problems into the 3D path.

A 3D mesh with the same bands, ny, and nz z-layers (periodic z), with w = 0
and z-constant data, reproduces the 2D reference on every z layer
(SURVEY §0.5, §7).  Variables map (rho, rho v1, rho v2, rho E) <- 3D
(0, 1, 2, 4); 3D variable 3 (rho w) must stay at rounding level.
"""
import numpy as np

from paper_2008_04356_b200 import types as T


def mesh3d(bands, ny, nz=1, periodic_x=True, width=2.0, height=2.0, depth=1.0):
    return T.mesh_spec(bands, ny=ny, nz=nz, width=width, height=height, depth=depth,
                       periodic=(periodic_x, True, True))


def case3d(case):
    if case == "density_wave":
        return T.density_wave(alpha=0.1, a=(1.0, 1.0, 0.0), k=(1.0, 1.0, 0.0), p0=1.0)
    if case == "freestream":
        return T.freestream(rho=1.0, v=(1.0, 0.5, 0.0), p=1.0)
    raise ValueError(case)


def layers(u3, bands, ny, nz, n):
    """3D field -> list of nz 2D fields (gid order of the 2D reference)."""
    ne2 = sum(b[0] for b in bands) * ny
    U3 = np.asarray(u3).reshape(-1, n, n, n, 5)
    out = []
    for iz in range(nz):
        L = np.zeros((ne2, n, n, 4))
        g2 = g3 = 0
        for nx, _, _ in bands:
            for ix in range(nx):
                for iy in range(ny):
                    L[g2 + ix * ny + iy] = U3[g3 + (ix * ny + iy) * nz + iz][:, :, iz if False else 0][..., [0, 1, 2, 4]]
            g2 += nx * ny
            g3 += nx * ny * nz
        out.append(L.reshape(-1))
    return out


def w_component(u3):
    return np.asarray(u3).reshape(-1, 5)[:, 3]


def max_layer_diff(u3, u2, bands, ny, nz, n):
    return max(np.abs(L - u2).max() for L in layers(u3, bands, ny, nz, n))

"""One configs[1] interface (16 x 16 faces against 12 x 12, N = 7, displaced by
(0.37, 0.11) t at t = 1.3): lifting mean and viscous interface flux on the device,
for an ncu launch list of the non-matching mortar kernels."""
import numpy as np

from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T

degree, n = 7, 8
nfy = nfz = [16, 12]
rng = np.random.default_rng(1)
u = []
for s in (0, 1):
    shape = (nfy[s], nfz[s], n, n)
    rho = 1.0 + 0.1 * rng.uniform(-1, 1, shape)
    st = np.zeros(shape + (5,))
    st[..., 0] = rho
    st[..., 1] = 0.3 * rho
    st[..., 4] = 1.0 / 0.4 + 0.5 * 0.09 * rho
    u.append(st)
g = [0.1 * rng.standard_normal((nfy[s], nfz[s], n, n, 12)) for s in (0, 1)]
gas = T.Gas(1.4, 287.0, 1e-3, 0.72)
for _ in range(2):
    capi.interface_lift_device(gas, degree, T.NODES_GAUSS, nfy, nfz, 0.125, 0.125, 0.481, 0.143, u[0], u[1])
    capi.interface_flux_device(gas, degree, T.NODES_GAUSS, nfy, nfz, 0.125, 0.125, 0.481, 0.143, u[0], u[1], g[0], g[1])
print("ok")

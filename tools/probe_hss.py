import sys; sys.path.insert(0, 'oracle/build'); sys.path.insert(0, 'tests')
import numpy as np
import _oracle as o
import paper_1611_01391_b200 as s
from hss_inputs import cauchy_kernel
M = cauchy_kernel(1024)
def run(lib, B, rho, seed):
    try:
        if lib is o:
            c = lib.cross_approx(B, rho, rho, rho, [], 2, 1.1, None, lib.Rng(seed))
        else:
            c = lib.cross_approx(B, rho, rho, rho, [], 2, 1.1, lib.Rng(seed))
        c = c[0] if isinstance(c, tuple) else c
        C = B[:, c['J']] @ c['nucleus'] @ B[c['I'], :]
        return c['I'], c['J'], np.linalg.norm(B - C) / np.linalg.norm(B)
    except Exception as e:
        return type(e).__name__ + ':' + str(e)[:60]
for name, B in (("cauchy512", np.asfortranarray(M[0:512, 512:1024])), ("cauchy256", np.asfortranarray(M[0:256, 256:512])),
                ("fg512", o.gen_factor_gaussian(512, 512, 8, 1e-9, o.Rng(3))), ("fg300", o.gen_factor_gaussian(300, 300, 8, 1e-9, o.Rng(3))),
                ("fg257", o.gen_factor_gaussian(257, 257, 8, 1e-9, o.Rng(3)))):
    for rho in (3, 6, 8):
        p, q = run(s, B, rho, 1), run(o, B, rho, 1)
        same = (p[0] == q[0] and p[1] == q[1]) if isinstance(p, tuple) and isinstance(q, tuple) else None
        print(name, rho, same, p if not isinstance(p, tuple) else p[2], q if not isinstance(q, tuple) else q[2])

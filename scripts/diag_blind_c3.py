"""Diagnostic: where the float32 error of one blind sweep (config 3) sits,
against the compiled reference and the float32 restatement floor."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import od2p as O, ref_lib as R
from tests import config_cases as CC
from tests.helpers import rel_l2
import paper_2011_00162_b200 as P

c = CC.case(3)
g = O.make_raster_scan(c.N_rows, c.N_cols, c.cfg.s, c.cfg.step)
oplan = O.plan_grid(g, *c.plan_kind[1:])
ref = R.blind_steps(c.ref_plan(), c.f, R.blind_cfg(**c.cfg.solver), 1, w0=c.w0)
fl = O.BlindSolver(oplan, c.f, O.BlindConfig(**c.cfg.solver), precision='f32')
fst = fl.init_state(c.w0); fl.step(fst)
gs = P.BlindSolver(c.gpu_plan(), c.f, P.BlindConfig(**c.cfg.solver), dtype='f32')
st = gs.init_state(c.w0); gs.step(st)
for k in ['w', 'w_copies', 'u', 'z', 'gamma']:
    a, b, r = getattr(st, k), getattr(fst, k), ref[k]
    if k == 'w':
        print(k, 'gpu %.3e floor %.3e' % (rel_l2(a, r), rel_l2(b, r)))
    else:
        print(k, 'gpu %.3e floor %.3e' % (max(rel_l2(x, y) for x, y in zip(a, r)), max(rel_l2(x, y) for x, y in zip(b, r))))
# forward of the disk: GPU op vs numpy f32 vs f64
gl = P.make_raster_scan(64, 64, 64, 16)
one = np.ones((64, 64), complex)
f64 = O.fft2n(c.w0)
print('fft(disk) gpu f32 %.3e numpy f32 %.3e' % (rel_l2(P.forward(c.w0, one, gl, dtype='f32')[0], f64),
                                                rel_l2(O.fft2n(c.w0.astype(np.complex64)), f64)))
# error location of z on subdomain 0
zr, zg, zf = ref['z'][0], st.z[0], fst.z[0]
y = ref['gamma'][0] + zr  # y = Gamma' + z
ay = np.abs(y)
for lo, hi in [(0, 1e-3), (1e-3, 1e-1), (1e-1, 1e1), (1e1, 1e9)]:
    m = (ay >= lo) & (ay < hi)
    print('|y| in [%g,%g): %d px, gpu err^2 share %.3f, floor err^2 share %.3f' % (
        lo, hi, m.sum(), np.sum(np.abs(zg - zr)[m] ** 2) / np.sum(np.abs(zg - zr) ** 2),
        np.sum(np.abs(zf - zr)[m] ** 2) / np.sum(np.abs(zf - zr) ** 2)))
# u error location vs density
ur, ug = ref['u'][0], st.u[0]
e = np.abs(ug - ur) ** 2
print('u err^2 share in the outer 32 px frame: %.3f' % (1 - e[32:-32, 32:-32].sum() / e.sum()))

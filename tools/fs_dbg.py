import sys, numpy as np
sys.path.insert(0, '.')
import paper_1205_4139_b200 as fmp
from oracle import Oracle
o = Oracle('restatement')
n, m = 1 << 18, 1 << 15
om = o.make_row_selection(n, m, 7 + n)
print('building op', flush=True)
op = fmp.SensingOperator('fourier', n, om)
print('op ok', flush=True)
r = o.rng_complex_gaussian(5, m)
h = op.apply_adjoint(r[None])[0]
want = o.apply_adjoint('fourier', n, om, r)
print('rel', np.linalg.norm(h - want) / np.linalg.norm(want), flush=True)

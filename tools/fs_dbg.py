import sys, numpy as np
sys.path.insert(0, '.')
import paper_1205_4139_b200 as fmp
from oracle import Oracle
o = Oracle('restatement')
n, m = 1 << 18, 1 << 15
om = o.make_row_selection(n, m, 7 + n)
for kind in ('fourier', 'hadamard'):
    op = fmp.SensingOperator(kind, n, om)
    r = o.rng_complex_gaussian(5, m)
    want = o.apply_adjoint(kind, n, om, r)
    for dt in (np.complex128, np.complex64):
        h = op.apply_adjoint(r.astype(dt)[None])[0]
        print(kind, np.dtype(dt).name, 'rel', np.linalg.norm(h - want) / np.linalg.norm(want), 'nz', np.count_nonzero(h), flush=True)
    x = o.rng_complex_gaussian(6, n)
    f = op.forward(x[None])[0]
    print(kind, 'forward rel', np.linalg.norm(f - o.forward(kind, x)) / np.linalg.norm(x), flush=True)

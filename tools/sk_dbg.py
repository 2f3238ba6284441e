import sys; sys.path[:0]=['tests','oracle','.']
import numpy as np
from helpers import load, device_cost, rel_err
from paper_2511_11359_b200 import sinkhorn as SK
d = load('sinkhorn_explicit_n37'); k = device_cost(d)
for eta, tol, mi in ((0.05, 1e-9, 10000), (0.01, 1e-8, 20000), (0.01, 1e-12, 7)):
    tag = f"eta{eta}_mi{mi}"
    pot = SK.sinkhorn_solve(k, d['r'], d['c'], eta, tol=tol, max_iter=mi)
    print(tag, pot.converged, pot.sweeps, pot.col_gap, d[f'{tag}_info'], rel_err(pot.phi, d[f'{tag}_phi']), rel_err(pot.psi, d[f'{tag}_psi']))
    print('dual', SK.eot_dual_value(pot, k, d['r'], d['c']), float(d[f'{tag}_dual']))
    print('col', rel_err(SK.sinkhorn_column_marginal(pot, k), d[f'{tag}_col']))

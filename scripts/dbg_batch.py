import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1805_08846_b200 as P
import cases
r = dict(cases.RECIPES["advection_square_7"])
print(r)
res = {}
for dc in (False, True):
    sim, g = cases.product_sim(r, device_controller=dc)
    rep = sim.run_until(1e30, max_steps=int(sys.argv[1]))
    res[dc] = (sim.grid.interior().copy(), [(a.dt, a.max_speed, a.accepted) for a in rep.attempts], sim._cur, sim._scratch)
    # raw buffers
    res[dc] += ([sim.device_grid.download(b) for b in range(3)],)
    sim.close()
h, d = res[False], res[True]
print('attempts', h[1], d[1])
print('cur', h[2], h[3], d[2], d[3])
print('diff idx', np.nonzero(h[0] != d[0]))
print('host', h[0].ravel()[:20])
print('dev ', d[0].ravel()[:20])
for b in range(3):
    print('buf', b, np.array_equal(h[4][b], d[4][b]), d[4][b].ravel()[:12])

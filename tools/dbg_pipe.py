import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import oracle as O
import paper_2405_16788_b200 as P
rng = np.random.default_rng(77)
n, C, q = 20000, 49, 600_000
pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
nrm = rng.standard_normal((n, 3)); nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
area = rng.uniform(0.5, 1, n) / n
mu = rng.standard_normal((n, C))
kinds = np.ones(C, np.uint8); kinds[0] = 0
t = P.DipoleTree(0); t.build(P.OrientedPointCloud(pos, nrm, area, mu)); t.set_channel_kernels(kinds)
xs = rng.uniform(-1.2, 1.2, (q, 3)).astype(np.float32).astype(np.float64)
p = P.KernelParams(epsilon=0.02)
host = t.primal(xs, p, 2.0)
dev = t.primal(torch.from_numpy(xs).cuda(), p, 2.0).cpu().numpy()
d = np.abs(host - dev)
print('max abs', d.max(), 'max rel', (d / (np.abs(dev) + 1e-30)).max(), 'scale', np.abs(dev).max())
bad = np.argwhere(d > 1e-9 + 1e-6 * np.abs(dev))
print('nbad', len(bad), bad[:5])
r = O.OracleTree(O.Cloud(pos, nrm, area, mu)); r.set_kinds(kinds)
idx = np.unique(np.concatenate([bad[:200, 0], np.arange(200)]))
want = r.primal(O.Params(0.02), 2.0, xs[idx])
for name, v in (('host', host), ('dev', dev)):
    e = np.abs(v[idx] - want)
    print(name, 'vs oracle max abs', e.max(), 'nbad(1e-4 rel,1e-6 abs)', int((e > 1e-6 + 1e-4 * np.abs(want)).sum()))

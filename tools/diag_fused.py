"""Diagnostic: fused batched factor + solve vs the oracle on sampled members of a batch."""
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402

n, k, B = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 100, 1024)
off = int(sys.argv[4]) if len(sys.argv) > 4 else 0
fused = not (len(sys.argv) > 5 and sys.argv[5] == "factor")
data = np.stack([generate_spd(n, k, off + s).data for s in range(B)])
rhs = np.stack([make_rhs(n, off + s) for s in range(B)])
a0, b0 = data.copy(), rhs.copy()
if fused:
    bc.factor_solve_batched(data, rhs, n, k)
else:
    bc.factor_batched(data, n, k)
    rhs = np.stack([bc.solve_with_factor(bc.BandedMatrix(n, k, None, data[s].copy()), b0[s]) for s in range(B)])
res = []
for s in sorted(set([0, 1, 2, B // 3, B // 2, B - 2, B - 1] + list(range(290, 300)) + list(range(min(B, 8))))):
    if s >= B:
        continue
    want = a0[s].copy()
    oracle.factor_plain(n, k, k + 1, want)
    el = oracle.max_scaled_diff(n, k, data[s], k + 1, want, k + 1)
    dl = np.abs(data[s] - want).reshape(n, k + 1) / np.maximum(np.abs(want).reshape(n, k + 1), 1)
    badc = np.nonzero(dl.max(axis=1) > 1e-10)[0]
    if len(badc):
        c0 = int(badc[0])
        offs = np.nonzero(dl[c0] > 1e-10)[0][:20]
        print("matrix", s, "first bad column", c0, "offsets", offs.tolist(), "n bad cols", len(badc), flush=True)
        gpu = data[s].reshape(n, k + 1)[c0, offs[:4]]
        ref = want.reshape(n, k + 1)[c0, offs[:4]]
        inp = a0[s].reshape(n, k + 1)[c0, offs[:4]]
        later = [a0[s].reshape(n, k + 1)[c0 + k + 16, offs[:4]]] if c0 + k + 16 < n else []
        print("   gpu", gpu, "ref", ref, "input", inp, "col+116 input", later, flush=True)
    xs = oracle.solve(n, k, k + 1, want, b0[s])
    err = np.abs(rhs[s] - xs)
    tol = 1e-8 * np.abs(xs).max()
    first = int(np.argmax(err > tol)) if (err > tol).any() else -1
    res.append((s, f"{el:.1e}", f"{err.max():.1e}", first))
print(n, k, B, res, flush=True)

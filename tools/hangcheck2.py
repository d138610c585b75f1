"""Factor the given shapes one at a time (n,k,ld triples), printing each before it runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402

for arg in sys.argv[1:]:
    n, k, ld = map(int, arg.split(","))
    print("run", n, k, ld, flush=True)
    a0 = bc.generate_spd(n, k, seed=1)
    a = bc.BandedMatrix(n, k, ld)
    a.data.reshape(n, ld)[:, :k + 1] = a0.data.reshape(n, k + 1)
    ref = a.copy()
    oracle.factor_plain(n, k, ld, ref.data)
    bc.factor_blocked_serial(a)
    err = oracle.max_scaled_diff(n, k, a.data, ld, ref.data, ld)
    print("  ok" if err <= 1e-10 else f"  BAD {err}", flush=True)
print("done")

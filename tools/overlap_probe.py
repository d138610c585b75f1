"""Does the backward sweep of one part of a C5 batch overlap the factorization tail of the next?
Splits the batch over P stream pairs: stream p runs fused-factor(part p) then backward(part p);
parts are launched in order, so part p's sweep gets the SM slots part p+1's factorization leaves."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402

n, k, batch = 4096, 100, 1024
a = np.stack([generate_spd(n, k, s).data for s in range(8)])
a0 = torch.from_numpy(np.concatenate([a] * (batch // 8))).cuda()
b0 = torch.from_numpy(np.stack([make_rhs(n, s) for s in range(batch)])).cuda()
w, wb, y = a0.clone(), b0.clone(), torch.empty_like(b0)
info = torch.zeros(batch, dtype=torch.int32, device="cuda")
main = torch.cuda.current_stream()


def run(parts):
    bounds = np.linspace(0, batch, len(parts) + 1).astype(int) if isinstance(parts, list) else None
    cuts = [0] + list(np.cumsum(parts)) if bounds is None else bounds
    streams = [torch.cuda.Stream() for _ in range(len(cuts) - 1)]
    w.copy_(a0); wb.copy_(b0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for p, st in enumerate(streams):
        lo, hi = int(cuts[p]), int(cuts[p + 1])
        st.wait_stream(main)
        with torch.cuda.stream(st):
            bc.dpbtrf_fwd_batched_device(w[lo:hi].view(-1), n, k, k + 1, wb[lo:hi].view(-1), y[lo:hi].view(-1),
                                         hi - lo, info=info[lo:hi], stream=st)
    for p, st in enumerate(streams):
        lo, hi = int(cuts[p]), int(cuts[p + 1])
        with torch.cuda.stream(st):
            bc.dpbtrs_bwd_batched_device(w[lo:hi].view(-1), n, k, k + 1, y[lo:hi].view(-1), wb[lo:hi].view(-1),
                                         hi - lo, info[lo:hi], stream=st)
    for st in streams:
        main.wait_stream(st)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for parts in ([1024], [512, 512], [888, 136], [592, 432], [296, 296, 296, 136], [740, 284], [256] * 4):
    ts = [run(parts) for _ in range(4)]
    print(parts, "ms", round(min(ts), 3), flush=True)
assert int(info.abs().sum().item()) == 0

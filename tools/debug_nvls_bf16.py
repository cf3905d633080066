import sys; sys.path.insert(0, '.')
import numpy as np, torch
import oracle
from tests import harness
from paper_2408_05962_b200 import hiccl as H
p = min(torch.cuda.device_count(), 4)
d = 1 << 16
for dtype in ("bf16", "f16", "f32"):
    plan, _, _ = harness.make_plan(7, 1, p, d, 0, 0, [p], p, 1, 1, 1)
    flat = oracle.FlatPlan.from_dicts(p, plan.buffers, plan.transfer_dicts())
    want = harness.run_oracle(flat, plan, dtype, 77)
    got, stats = harness.run_device(plan, dtype, 77, devices=tuple(range(p)), nvls=True)
    sends = harness.initial_state(plan, dtype, 77)["sendbuf"]
    def f64(a):
        if dtype == "bf16": return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        if dtype == "f16": return a.view(np.float16).astype(np.float64)
        return a.astype(np.float64)
    exact = np.sum([f64(s) for s in sends], axis=0)
    mag = np.sum([np.abs(f64(s)) for s in sends], axis=0)
    for r in range(p):
        g = f64(got["recvbuf"][r]); w = f64(want["recvbuf"][r])
        rel = np.abs(g - w) / mag
        bad = np.nonzero(rel > 1e-2)[0]
        print(dtype, "rank", r, "bad", bad.size, "max rel", rel.max(), "first", bad[:8], "chunk", bad[:8] // d if bad.size else None)
        for i in bad[:4]:
            print("   i", i, "got", g[i], "want", w[i], "exact", exact[i], "mag", mag[i], [f64(s)[i] for s in sends])
        same = (got["recvbuf"][r] == got["recvbuf"][0]).all()
        print("   identical to rank0:", same, "g vs exact maxrel", (np.abs(g - exact) / mag).max())

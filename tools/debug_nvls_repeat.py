import sys; sys.path.insert(0, '.')
import numpy as np, torch
from tests import harness
p = min(torch.cuda.device_count(), 4)
d = 1 << 16
fails = {}
for it in range(12):
    for kind, form in [(7, 2), (7, 1), (5, 0), (6, 0)]:
        plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 1)
        got, stats = harness.run_device(plan, "f32", 77 + it, devices=tuple(range(p)), nvls=True)
        st = harness.initial_state(plan, "f32", 77 + it)
        if kind == 5:
            want = [np.concatenate(st["sendbuf"]) for _ in range(p)]
            bad = [int((got["recvbuf"][r] != want[r]).sum()) for r in range(p)]
        else:
            exact = harness.exact_reduction(kind, p, d, 0, "f32", st["sendbuf"], st["recvbuf"])
            mag = np.sum([np.abs(s.astype(np.float64)) for s in st["sendbuf"]], axis=0)
            bad = [int((np.abs(got["recvbuf"][r].astype(np.float64) - exact["recvbuf"][r]) > 1e-6 * mag).sum()) for r in range(p)]
        if any(bad):
            fails.setdefault((kind, form), []).append((it, bad))
print("fails", fails)

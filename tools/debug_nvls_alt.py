import sys; sys.path.insert(0, '.')
import numpy as np, torch
import oracle
from tests import harness
p = min(torch.cuda.device_count(), 4)
d = 1 << 16
for kind, form in [(7, 2), (7, 1), (3, 0)]:
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 1)
    got, stats = harness.run_device(plan, "f32", 77, devices=tuple(range(p)), nvls=True)
    st = harness.initial_state(plan, "f32", 77)
    exact = harness.exact_reduction(kind, p, d, 0, "f32", st["sendbuf"], st["recvbuf"])
    mag = np.sum([np.abs(s.astype(np.float64)) for s in st["sendbuf"]], axis=0)
    print(kind, form, "nvls items", [s["nvls_items"] for s in stats], "items", [s["num_items"] for s in stats])
    for r in range(p):
        g = got["recvbuf"][r].astype(np.float64)
        w = exact["recvbuf"][r]
        rel = np.abs(g - w) / mag
        bad = np.nonzero(rel > 1e-6)[0]
        print("  rank", r, "bad", bad.size, "first", bad[:5], "max rel", rel.max())
        for i in bad[:3]:
            print("     i", i, "got", g[i], "exact", w[i], "init", st["recvbuf"][r][i])

"""Small, repeatable executor launches for ncu (development tool).

  python tools/profile_target.py [ar1|ar8v|ag8v] [--mib N]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_05962_b200 import hiccl as H

which = sys.argv[1] if len(sys.argv) > 1 else "ar1"
mib = int(sys.argv[sys.argv.index("--mib") + 1]) if "--mib" in sys.argv else 1024
S = mib << 20
cfg = {"ar1": (7, 0, 1, [1], 1), "ar8v": (7, 1, 8, [8], 8), "ag8v": (5, 0, 8, [8], 8),
       "ar8v24": (7, 1, 8, [2, 4], 4)}[which]
kind, form, p, hier, g = cfg
d = S // (4 * p)
spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), 0, d)
plan = H.lower(H.build(spec, p), H.Machine(hier, g))
w = H.World(plan, [0], "f32")
sl, rl = H.preset_lengths(spec, p)
keep = []
for r in range(p):
    for name, n in (("sendbuf", sl), ("recvbuf", rl)):
        t = torch.zeros(n * 4, dtype=torch.uint8, device="cuda:0")
        keep.append(t)
        w.bind(r, name, t.data_ptr(), t.numel())
w.commit()
for _ in range(4):
    w.run()
torch.cuda.synchronize()
print("ok", which, mib, "MiB", w.execs[0].stats())

"""Small, repeatable executor launches for ncu (development tool).

  python tools/profile_target.py [ar1|ar8v|ag8v|ar8v24|c1] [--mib N]

c1 = BASELINE config C1 as bench.py's virtual_c1 leg runs it: all-reduce
multi, p=8 on the virtual {2,4} (g=4), stripe 4, ring 2, pipeline 4.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_05962_b200 import hiccl as H

which = sys.argv[1] if len(sys.argv) > 1 else "ar1"
mib = int(sys.argv[sys.argv.index("--mib") + 1]) if "--mib" in sys.argv else 1024
S = mib << 20
cfgs = {"ar1": (7, 0, 1, [1], 1), "ar8v": (7, 1, 8, [8], 8), "ag8v": (5, 0, 8, [8], 8),
        "ar8v24": (7, 1, 8, [2, 4], 4)}
if which == "c1":
    cfg, ring, stripe, pipe = (7, 1, 8, [2, 4], 4), 2, 4, 4
    S = (mib if "--mib" in sys.argv else 64) << 20
else:
    cfg, ring, stripe, pipe = cfgs[which], 1, 1, 1
kind, form, p, hier, g = cfg
d = S // (4 * p)
spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), 0, d)
plan = H.lower(H.build(spec, p), H.Machine(hier, g), ring=ring, stripe=stripe, pipeline=pipe)
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
if "--time" in sys.argv:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        w.start()
    b.record()
    w.wait()
    torch.cuda.synchronize()
    print(f"{which}: {a.elapsed_time(b) / 20 * 1e3:.1f} us per launch")
print("ok", which, mib, "MiB", w.execs[0].stats())
if "--trace" in sys.argv:
    # device timeline of the last launch (CTA 0's step publishes) beside
    # each step's algorithmic bytes (sources read once + one store)
    import json
    w.run()
    torch.cuda.synchronize()
    tr = w.execs[0].trace()
    summ = plan.schedule_summary(num_execs=1, copy_mode="push", verify=False)
    per = [0] * summ["steps"]
    for it in summ["item_list"]:
        per[it["step"]] += (it["n_src"] + 1) * it["count"] * 4
    lay = plan.layout_summary(num_execs=1)["execs"][0]
    prev = tr["entry_barrier_us"] or 0.0
    for s, t in enumerate(tr["steps_us"]):
        dt = (t or 0.0) - prev
        print(json.dumps({"step": s, "end_us": t, "dur_us": round(dt, 1), "bytes": per[s],
                          "gbs": round(per[s] / max(dt, 1e-3) / 1e3, 1),
                          "tiles": lay["tiles"][s], "cta_peak_tiles": lay["cta_peak_tiles"][s]}))
        prev = t or prev
    print(json.dumps({"last_cta_us": tr["last_cta_us"], "exit_us": tr["exit_us"]}))

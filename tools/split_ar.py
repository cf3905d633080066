"""Development experiment: one all-reduce split between the NVLS library and
point to point, both halves in the same launch (same steps, disjoint
buffers): does the switch path leave link capacity the point-to-point path
can use?

  python tools/split_ar.py [--mib 1024] [--fractions 0,0.5,0.6,0.7,1]

A custom composition (the paper's API): reduce-scatter + in-place
all-gather of buffers A (fraction f of the elements, in the NVLS window)
and B (the rest, ordinary device memory), one process driving every GPU.
Prints us per launch and busbw for each f; results are checked against the
exact sum.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_05962_b200 import hiccl as H  # noqa: E402


def program(p: int, na: int, nb: int) -> H.CollectiveProgram:
    prog = H.CollectiveProgram(p)
    parts = [(x, n) for x, n in (("A", na), ("B", nb)) if n]
    for x, n in parts:
        prog.declare_buffer("s" + x, p * n, input=True).declare_buffer("r" + x, p * n)
    for x, n in parts:
        for j in range(p):
            prog.add_reduction(H.BufferRef("s" + x, j * n, n), H.BufferRef("r" + x, j * n, n),
                               list(range(p)), j)
    prog.add_fence()
    for x, n in parts:
        for i in range(p):
            prog.add_multicast(H.BufferRef("r" + x, i * n, n), H.BufferRef("r" + x, i * n, n), i,
                               [r for r in range(p) if r != i])
    return prog


def run(p: int, S: int, f: float, iters: int = 20):
    d = S // (4 * p)  # elements per chunk in total
    na = int(d * f) // 1024 * 1024
    nb = d - na
    plan = H.lower(program(p, na, nb), H.Machine([p], p))
    devs = list(range(p))
    world = H.World(plan, devs, "f32", copy_mode="push")
    keep = []
    ptrs = {}
    if na:
        where = world.enable_nvls({"sA": p * na * 4, "rA": p * na * 4})
        for (r, name), ptr in where.items():
            ptrs[(r, name)] = ptr
    if nb:
        for r in range(p):
            for name in ("sB", "rB"):
                t = torch.zeros(p * nb * 4, dtype=torch.uint8, device=f"cuda:{r}")
                keep.append(t)
                world.bind(r, name, t.data_ptr(), t.numel())
                ptrs[(r, name)] = t.data_ptr()
    for r in range(p):
        for x, n in (("A", na), ("B", nb)):
            if n:
                H.device_fill(r, ptrs[(r, "s" + x)], p * n, "f32", 7, r)
    world.commit()
    for dv in devs:
        torch.cuda.synchronize(dv)
    for _ in range(3):
        world.run()
    streams = [torch.cuda.Stream(dv) for dv in devs]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in devs]
    for i, dv in enumerate(devs):
        with torch.cuda.device(dv):
            ev[i][0].record(streams[i])
    for _ in range(iters):
        world.start([s.cuda_stream for s in streams])
    for i, dv in enumerate(devs):
        with torch.cuda.device(dv):
            ev[i][1].record(streams[i])
    world.wait()
    for dv in devs:
        torch.cuda.synchronize(dv)
    t = max(a.elapsed_time(b) for a, b in ev) / iters / 1e3
    # spot check: element 0..4095 of each part against the fp64 sum
    ok = True
    for x, n in (("A", na), ("B", nb)):
        if not n:
            continue
        m = min(4096, p * n)
        exact = np.zeros(m)
        for r in range(p):
            tmp = torch.empty(m, dtype=torch.float32, device="cuda:0")
            H.device_fill(0, tmp.data_ptr(), m, "f32", 7, r)
            exact += tmp.cpu().numpy().astype(np.float64)
        got = torch.empty(m * 4, dtype=torch.uint8, device="cuda:0")
        src = torch.as_tensor(H.DeviceView(ptrs[(0, "r" + x)], m * 4), device="cuda:0") \
            if x == "A" else None
        if src is None:
            got = [k for k in keep if k.data_ptr() == ptrs[(0, "rB")]][0][: m * 4]
        else:
            got.copy_(src)
        g = got.cpu().numpy().view(np.float32).astype(np.float64)
        ok &= bool(np.max(np.abs(g - exact)) < 1e-4)
    world.close()
    alg = S / t / 1e9
    return {"f_nvls": round(na / d, 3), "us": round(t * 1e6, 1), "algbw": round(alg, 1),
            "busbw": round(alg * 2 * (p - 1) / p, 1), "ok": ok}


def main():
    mib = int(sys.argv[sys.argv.index("--mib") + 1]) if "--mib" in sys.argv else 1024
    fr = [float(x) for x in (sys.argv[sys.argv.index("--fractions") + 1].split(",")
                             if "--fractions" in sys.argv else "0,0.5,0.6,0.7,0.8,1".split(","))]
    p = torch.cuda.device_count()
    for f in fr:
        print(json.dumps({"p": p, "mib": mib, **run(p, mib << 20, f)}), flush=True)


if __name__ == "__main__":
    main()

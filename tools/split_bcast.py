"""Development experiment: one broadcast from rank 0 split between the NVLS
library (multimem.st from the root, issue-limited near 570 GB/s) and a
pipelined point-to-point chain 0 -> 1 -> ... -> p-1, both in the same
launch: does the chain use the root link capacity the multicast leaves?

  python tools/split_bcast.py [--mib 1024] [--m 32] [--fractions 0,0.3,0.5,1]

A custom composition (the paper's API), one process driving every GPU:
buffer A (fraction f, in the NVLS window) goes out chunk by chunk as in-place
every-rank multicasts (lowered to multimem.st), buffer B (the rest) as a
chain, chunk c taking hop h in step c + h. Prints us per launch and GB/s;
every rank's result is compared with the root's input.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2408_05962_b200 import hiccl as H  # noqa: E402


def program(p: int, na: int, nb: int, m: int) -> H.CollectiveProgram:
    prog = H.CollectiveProgram(p)
    if na:
        prog.declare_buffer("A", na, input=True)
    if nb:
        prog.declare_buffer("B", nb, input=True)
    ca, cb = -(-na // m), -(-nb // m)
    nsteps = max(m if na else 0, (m + p - 2) if nb else 0)
    for s in range(nsteps):
        if s:
            prog.add_fence()
        if na and s < m and s * ca < na:
            off = s * ca
            n = min(ca, na - off)
            prog.add_multicast(H.BufferRef("A", off, n), H.BufferRef("A", off, n), 0,
                               list(range(1, p)))
        if nb:
            for h in range(p - 1):
                c = s - h
                if 0 <= c < m and c * cb < nb:
                    off = c * cb
                    n = min(cb, nb - off)
                    prog.add_multicast(H.BufferRef("B", off, n), H.BufferRef("B", off, n), h,
                                       [h + 1])
    return prog


def run(p: int, S: int, f: float, m: int, iters: int = 10):
    d = S // 4
    na = int(d * f) // (1024 * m) * (1024 * m)
    nb = d - na
    plan = H.lower(program(p, na, nb, m), H.Machine([p], p))
    devs = list(range(p))
    world = H.World(plan, devs, "f32", copy_mode="push")
    keep, ptrs = [], {}
    if na:
        ptrs.update(world.enable_nvls({"A": na * 4}))
    if nb:
        for r in range(p):
            t = torch.zeros(nb * 4, dtype=torch.uint8, device=f"cuda:{r}")
            keep.append(t)
            world.bind(r, "B", t.data_ptr(), t.numel())
            ptrs[(r, "B")] = t.data_ptr()
    parts = [(x, n) for x, n in (("A", na), ("B", nb)) if n]
    for x, n in parts:
        H.device_fill(0, ptrs[(0, x)], n, "f32", 7, 0)
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
    ok = True
    for x, n in parts:
        want = torch.as_tensor(H.DeviceView(ptrs[(0, x)], n * 4), device="cuda:0").cpu()
        for r in range(1, p):
            got = torch.as_tensor(H.DeviceView(ptrs[(r, x)], n * 4), device=f"cuda:{r}").cpu()
            ok &= bool(torch.equal(got, want))
    world.close()
    return {"f_nvls": round(na / d, 3), "m": m, "us": round(t * 1e6, 1),
            "algbw": round(S / t / 1e9, 1), "ok": ok}


def main():
    arg = lambda k, dflt: sys.argv[sys.argv.index(k) + 1] if k in sys.argv else dflt
    mib = int(arg("--mib", "1024"))
    m = int(arg("--m", "32"))
    fr = [float(x) for x in arg("--fractions", "0,0.3,0.5,0.7,1").split(",")]
    p = torch.cuda.device_count()
    for f in fr:
        print(json.dumps({"p": p, "mib": mib, **run(p, mib << 20, f, m)}), flush=True)


if __name__ == "__main__":
    main()

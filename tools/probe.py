"""Quick device-time probe of the executor on one GPU (development tool)."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2408_05962_b200 import hiccl as H

def probe(kind, form, p, S, hier=None, g=None, ring=1, stripe=1, m=1, dtype="f32", iters=10, **kw):
    esz = H.ELEMENT_SIZE[dtype]
    send_len, recv_len = H.preset_lengths(H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), 0, S // (esz * p)), p)
    d = S // (esz * p)
    spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), 0, d)
    plan = H.lower(H.build(spec, p), H.Machine(hier or [p], g or p), ring=ring, stripe=stripe, pipeline=m)
    w = H.World(plan, [0], dtype, **kw)
    keep = []
    for r in range(p):
        for name, n in (("sendbuf", send_len), ("recvbuf", recv_len)):
            t = torch.empty(n * esz, dtype=torch.uint8, device="cuda:0")
            keep.append(t)
            w.bind(r, name, t.data_ptr(), t.numel())
    w.commit()
    s = torch.cuda.Stream()
    for _ in range(3):
        w.execs[0].start(s.cuda_stream); w.execs[0].wait()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * iters)]
    for i in range(iters):
        evs[2*i].record(s)
        w.execs[0].start(s.cuda_stream)
        evs[2*i+1].record(s)
    torch.cuda.synchronize()
    ts = [evs[2*i].elapsed_time(evs[2*i+1]) for i in range(iters)]
    st = w.execs[0].stats()
    w.close()
    return min(ts), sum(ts)/len(ts), st

if __name__ == "__main__":
    GiB = 1 << 30
    a = torch.empty(GiB, dtype=torch.uint8, device="cuda:0"); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    print(f"torch copy 1GiB: {t:.3f} ms -> {2*GiB/t/1e6:.0f} GB/s r+w")
    del a, b
    for ctas, threads in [(0, 0), (148, 384), (148, 256), (296, 256), (296, 192), (444, 128), (592, 128)]:
        try:
            tmin, tavg, st = probe(7, 0, 1, GiB, ctas=ctas, threads=threads)
            print(f"AR p=1 1GiB ctas={st['ctas']} thr={st['threads']}: min {tmin:.3f} ms avg {tavg:.3f} -> {2*GiB/tmin/1e6:.0f} GB/s r+w")
        except Exception as e:
            print("fail", ctas, threads, e)
    for p in (8,):
        tmin, tavg, st = probe(7, 1, p, GiB // 8)
        print(f"AR multi p={p} 128MiB/rank virtual on 1 GPU: {tmin:.3f} ms; items {st['num_items']} steps {st['num_steps']}")

"""Host cost of Executor.start(): CPU time per call for a tiny plan (one
GPU, p = 1 and p = 8 virtual), and the device time per launch when
launches are issued back to back, against an empty torch kernel launch.

  python tools/launch_cost.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_05962_b200 import hiccl as H  # noqa: E402
from tests import harness  # noqa: E402


def measure(p, kind=7, form=1, d=256, mode="push", n=2000):
    plan, _, _ = harness.make_plan(kind, form, p, d, 0, 0, [p], p, 1, 1, 1)
    w = H.World(plan, [0], "f32", copy_mode=mode)
    keep = []
    for name, length, inp, internal in plan.buffers:
        if internal:
            continue
        for r in range(p):
            t = torch.zeros(length * 4, dtype=torch.uint8, device="cuda:0")
            keep.append(t)
            w.bind(r, name, t.data_ptr(), t.numel())
    w.commit()
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    for _ in range(50):
        w.start([sp])
    w.wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        w.start([sp])
    t1 = time.perf_counter()
    w.wait()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    w.close()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


def main():
    x = torch.zeros(1, device="cuda:0")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        x.add_(1)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"torch add_ launch: {(t1 - t0) / 2000 * 1e6:.2f} us CPU per call")
    for p, mode in ((1, "push"), (8, "push"), (8, "ll")):
        cpu, total = measure(p, mode=mode)
        print(f"p={p} {mode}: start() {cpu:.2f} us CPU per call, {total:.2f} us per launch end to end")


if __name__ == "__main__":
    main()

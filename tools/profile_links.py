"""One executor's NVLink traffic, measured by ncu.

ncu serializes kernels, and executors normally wait for each other (entry /
exit barriers, cross-executor step flags), so a multi-GPU launch cannot be
replayed. Schedules whose steps have no cross-executor wait (all-reduce
multi, all-gather and reduce-scatter single in push mode: every remote
access is a pull of an input or a push of a result) only need the barriers
for buffer reuse across launches; HICCL_PROFILE_SOLO=1 drops them, so each
executor's kernel runs (and replays) alone. The per-kernel counters

  nvltx__bytes.sum / nvlrx__bytes.sum   (link bytes, 32 B granularity)
  dram__bytes_read.sum / _write.sum     (HBM)

are then compared with the plan's comm_matrix bytes (pipeline.cpp:134-145).

  HICCL_PROFILE_SOLO=1 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,\
      nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:persistent --csv python tools/profile_links.py ar 4 --mib 256

prints the plan's expected per-GPU egress / ingress as a JSON line.
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2408_05962_b200 import hiccl as H  # noqa: E402

KINDS = {"ar": (7, 1), "ag": (5, 0), "rs": (6, 0)}


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "ar"
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    mib = int(sys.argv[sys.argv.index("--mib") + 1]) if "--mib" in sys.argv else 256
    kind, form = KINDS[which]
    assert os.environ.get("HICCL_PROFILE_SOLO") == "1", "set HICCL_PROFILE_SOLO=1"
    S = mib << 20
    d = S // (4 * p)
    spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), 0, d)
    plan = H.lower(H.build(spec, p), H.Machine([p], p))
    summ = plan.schedule_summary(num_execs=p, copy_mode="push", verify=False)
    assert all(e["remote_waits"] == 0 for e in summ["execs"]), "schedule has cross-executor waits"
    devs = list(range(p))
    world = H.World(plan, devs, "f32", copy_mode="push")
    sl, rl = H.preset_lengths(spec, p)
    keep = []
    nvls = "--nvls" in sys.argv  # buffers in a multicast window: multimem lowering
    if nvls:
        world.enable_nvls({"sendbuf": sl * 4, "recvbuf": rl * 4})
    else:
        for r in range(p):
            for name, n in (("sendbuf", sl), ("recvbuf", rl)):
                t = torch.zeros(n * 4, dtype=torch.uint8, device=f"cuda:{r}")
                keep.append(t)
                world.bind(r, name, t.data_ptr(), t.numel())
    world.commit()
    for _ in range(2):
        world.run()
    for dv in devs:
        torch.cuda.synchronize(dv)
    mat = [[0] * p for _ in range(p)]
    for slot in range(summ["steps"] + 4):
        try:
            m = plan.comm_matrix(slot)
        except H.HicclError:
            break
        for i in range(p):
            for j in range(p):
                mat[i][j] += m[i][j]
    egress = [sum(mat[i][j] for j in range(p) if j != i) for i in range(p)]
    ingress = [sum(mat[j][i] for j in range(p) if j != i) for i in range(p)]
    print(json.dumps({"collective": which, "p": p, "bytes_per_rank": S, "nvls": nvls,
                      "nvls_items": [e.stats()["nvls_items"] for e in world.execs],
                      "plan_egress_bytes": egress, "plan_ingress_bytes": ingress,
                      "launches_per_executor": 2}))
    world.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Headline benchmark: All-Reduce (and All-Gather) algbw on N B200s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hiccl|reference]
  torchrun --nproc-per-node N ... bench.py --gpus N      (N > 1, one rank per GPU)

Workload (BASELINE.json metric): All-Reduce, reduce-scatter +
all-gather formulation (presets.cpp:208-216), p = N ranks on the flat {N}
NVSwitch hierarchy, S = 1 GiB of fp32 per rank (sendbuf p*d elements), one
step = one start()/wait() of the persistent executor over the whole buffer.
Inputs are 1 GiB per rank (> 126 MB L2), so no L2 flush is needed between
steps. value = algbw = S / t (the reference's d*p/t, perf.cpp:137-140);
busbw = algbw * 2(p-1)/p. At N = 1 the plan is one local copy and the
roofline is HBM; at N > 1 it is NVLink (900 GB/s per direction nominal).

The reference arm (--impl reference) times the reference's own executor —
the symbolic execute_plan of the compiled reference library (oracle/_ref,
engine.cpp:285-347) — on bounded slices of the same workload, one worker
process per host core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GiB = 1 << 30
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
NVLINK_NOMINAL = 900.0
NVLINK_MEASURED_PEER = 770.0  # B200_PROFILING.md measured peer copy, per direction


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hiccl", choices=["hiccl", "reference"])
    ap.add_argument("--bytes", type=int, default=GiB, help="per-rank buffer S")
    ap.add_argument("--pipeline", type=int, default=1)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--copy-mode", default="push", choices=["pull", "push"])
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--nvls", default="auto", choices=["auto", "on", "off"],
                    help="all-reduce buffers in an NVSwitch multicast window (library NVLS: "
                         "fused multimem.ld_reduce + multimem.st per tile, S(1+1/p) per link "
                         "direction against 2S(p-1)/p point to point); auto = when the cost "
                         "model (hc_tune_nvls) predicts it faster")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e/nccl/all-gather/cpu legs")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers

def peaks() -> dict:
    try:
        return json.loads(PEAKS_FILE.read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every ~2 ms while
    the timed region runs (nvidia-smi's 100 ms loop would miss a short run)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.sm: list[float] = []
        self.max_sm = None
        self.reasons: set[str] = set()
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.ok = True
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception:
            self.ok = False
        return self

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                try:
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for name, bit in self.REASONS.items():
                    if bits & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0001)  # a 1 GiB copy step is ~0.33 ms: sample as often as NVML answers

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_sm,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "NVML"}


def bind_to_gpu_numa(device: int) -> list[int] | None:
    """Pin this process to the host cores NVML reports as close to `device`,
    so its pinned host buffers are allocated on the GPU's NUMA node (the
    e2e leg streams 2 GiB per step through them)."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(device)
        words = nv.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
        cpus = [c for c in cpus if c < (os.cpu_count() or 1)]
        if cpus:
            os.sched_setaffinity(0, cpus)
            return cpus
    except Exception:
        pass
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


# ------------------------------------------------------------------ reference arm

_REF = None


def _ref_worker_init():
    global _REF
    import oracle
    _REF = oracle.Reference()


def _ref_sample(job):
    """One bounded sample of the workload through the reference's executor
    (symbolic execute_plan, engine.cpp:285-347); returns its seconds."""
    p, d, m = job
    form = 1 if p > 1 else 0
    return _REF.time_execute_plan(7, form, p, d, 0, 0, [p], p, 1, 1, m)


def run_reference(args, world, rank):
    """Reference's own executor (symbolic execute_plan) on every host core:
    the all-reduce is elementwise, so the workload splits into independent
    slices, one per worker process, each run by the unmodified reference
    library (oracle/_ref, single-threaded by design)."""
    if rank != 0:
        return
    import oracle
    out = {"metric": "all_reduce_algbw", "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic"}
    p = args.gpus
    if not oracle.reference_available():
        out["unavailable"] = "oracle/_ref/libhiercoll_ref.so not built (needs /root/reference)"
        emit(out)
        return
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    # Bounded sample per worker: the symbolic engine keeps one provenance
    # object per element (~2.8 GB RSS per MiB/rank at p=8), so
    # slices stay small and the worker count is capped by host memory.
    slice_bytes = (4 << 20) if p == 1 else (1 << 20)
    d = max(1, slice_bytes // (4 * p))
    S = d * p * 4
    cores = os.cpu_count() or 1
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 16 << 30
    per_worker = max(256 << 20, int(3e9 * S / (1 << 20) * max(1, p) / 8))
    workers = max(1, min(cores, 64, int(avail * 0.5 // per_worker)))
    jobs = [(p, d, args.pipeline)] * workers
    # load the reference library here, in the parent, so the forked workers
    # inherit it (and the process that launched the arm has it mapped)
    _ref_worker_init()
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as pool:
        for _ in range(args.warmup):
            list(pool.map(_ref_sample, jobs))
        walls = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            list(pool.map(_ref_sample, jobs))
            walls.append(time.perf_counter() - t0)
    t = statistics.mean(walls)
    val = workers * S / t / 1e9
    out.update({"value": val, "ms_per_step": t * 1e3,
                "config": {"workload": f"all_reduce {'multi' if p > 1 else 'single'} p={p} flat "
                                       f"{{{p}}}, reference symbolic executor, {workers} slices of "
                                       f"{S} B/rank per step", "collective": "all_reduce",
                           "p": p, "bytes_per_rank": workers * S},
                "cpu_baseline": {"value": val, "unit": "GB/s", "cores": workers, "kind": "reference",
                                 "sample": f"{workers} independent slices of {S} B per rank (p={p}) "
                                           f"per step, each execute_plan of the reference library "
                                           f"in its own process (host wall clock)"},
                "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}})
    emit(out)


# ------------------------------------------------------------------ C1 on one GPU

def virtual_c1_leg(args, dev: int, all_cpus) -> dict:
    """BASELINE config C1 on one GPU: all-reduce multi, p = 8 ranks of the
    virtual {2,4} hierarchy (g = 4), stripe 4, ring 2, pipeline 4, 64 MiB of
    fp32 per rank — the fused executor (1,376 write groups, 9 steps), all
    eight ranks' buffers in this GPU's HBM, so the bound is HBM. Algorithmic
    bytes per launch = sum over the schedule's write groups of
    (sources + 1) x count x 4 (each source read once, one store), the same
    figure ncu's dram bytes are compared with. Checked bit for bit against
    the oracle replaying the same plan, which is also the leg's CPU
    baseline (whole plan, every host core)."""
    import numpy as np
    import torch
    from paper_2408_05962_b200 import hiccl as H

    p, d, dtype, esz = 8, 1 << 21, "f32", 4
    spec = H.CollectiveSpec(H.CollectiveKind.all_reduce, H.Formulation.multi, 0, d)
    plan = H.lower(H.build(spec, p), H.Machine([2, 4], 4), ring=2, stripe=4, pipeline=4)
    summ = plan.schedule_summary(num_execs=1, copy_mode="push", verify=False)
    alg = sum((it["n_src"] + 1) * it["count"] * esz for it in summ["item_list"])
    world = H.World(plan, [dev], dtype)
    # inputs from the product's device generator, outputs zeroed; the
    # oracle (below, after timing) starts from the same state
    tensors = {}
    for name, length, inp, internal in plan.buffers:
        if internal:
            continue
        for r in range(p):
            t = torch.zeros(length * esz, dtype=torch.uint8, device=f"cuda:{dev}")
            if inp:
                H.device_fill(dev, t.data_ptr(), length, dtype, 1234, r)
            world.bind(r, name, t.data_ptr(), t.numel())
            tensors[(name, r)] = t
    torch.cuda.synchronize(dev)
    world.commit()
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream
    for _ in range(max(3, args.warmup)):
        world.start([sp])
    world.wait()
    torch.cuda.synchronize(dev)
    steps = max(args.steps, 10)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        for k in range(steps):
            world.start([sp])
            ev[k + 1].record(stream)
    world.wait()
    torch.cuda.synchronize(dev)
    per = [ev[k].elapsed_time(ev[k + 1]) / 1e3 for k in range(steps)]
    t = ev[0].elapsed_time(ev[steps]) / 1e3 / steps
    names = sorted({name for name, _ in tensors})
    got = {name: [tensors[(name, r)].cpu().numpy().view(np.float32) for r in range(p)]
           for name in names}
    stats = world.execs[0].stats()
    world.close()
    del tensors
    torch.cuda.empty_cache()

    # checker and CPU baseline (test infrastructure, after the timed region):
    # the oracle replays the same plan on every host core
    import oracle
    os.sched_setaffinity(0, all_cpus)
    cores = len(all_cpus)
    flat = oracle.FlatPlan.from_dicts(plan.world_size, plan.buffers, plan.transfer_dicts())
    st = {name: [oracle.fill(length, dtype, 1234, r) if inp else np.zeros(length, np.float32)
                 for r in range(p)]
          for name, length, inp, internal in plan.buffers if not internal}
    t0 = time.perf_counter()
    oracle.execute(flat, dtype, st, threads=cores)
    tc = time.perf_counter() - t0
    exact = all(got[n][r].tobytes() == st[n][r].tobytes() for n in got for r in range(p))
    S = p * d * esz
    P = peaks()
    achieved = alg / statistics.mean(per) / 1e9
    tj = {}
    try:
        tj = json.loads((ROOT / "profiles" / "traffic.json").read_text())
    except Exception:
        pass
    return {"workload": "all_reduce multi p=8 virtual {2,4} g=4 stripe=4 ring=2 pipeline=4, "
                        "64 MiB fp32 per rank, 8 ranks on one GPU (BASELINE config C1)",
            "algbw": S / t / 1e9, "unit": "GB/s", "ms_per_step": t * 1e3, "steps": steps,
            "write_groups": len(summ["item_list"]), "device_steps": summ["steps"],
            "ctas": stats["ctas"], "threads": stats["threads"],
            "bitwise_vs_oracle": exact,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": P.get("hbm_gbs", 6650.0),
                         "unit": "GB/s", "frac": achieved / P.get("hbm_gbs", 6650.0),
                         "traffic": tj.get("virtual_c1_p8_2x4"),
                         "algorithmic_bytes_per_launch": alg,
                         "algorithmic_bytes_note": "sum over write groups of (sources + 1) x "
                                                   "count x 4 B: every source read once, one store"},
            "cpu_baseline": {"value": S / tc / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
                             "sample": "the whole C1 plan (64 MiB per rank, 8 ranks), "
                                       f"oracle/numeric_exec.c with {cores} threads, one run"}}


# ------------------------------------------------------------------ our arm

RESULT_OUT = sys.stdout


def emit(result: dict) -> None:
    RESULT_OUT.write(json.dumps(result) + "\n")
    RESULT_OUT.flush()


def respawn_under_torchrun(n: int) -> None:
    """`bench.py --gpus N` started by hand (no WORLD_SIZE): re-exec as N
    ranks through torch.distributed.run on this node, one process per GPU;
    rank 0 prints the line, so stdout carries exactly one JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    os.execvpe(sys.executable, cmd, env)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        respawn_under_torchrun(args.gpus)
    world, rank, local = dist_env()
    if world != args.gpus:
        sys.exit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # stdout carries exactly one JSON line: everything else that writes to
    # fd 1 (NCCL's version banner, library chatter) goes to stderr
    global RESULT_OUT
    RESULT_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        # rank 0 alone times the reference on the host; the others exit 0
        run_reference(args, world, rank)
        return
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist

    import numpy as np
    import torch
    from paper_2408_05962_b200 import hiccl as H
    from paper_2408_05962_b200.dist import DistCommunicator

    all_cpus = os.sched_getaffinity(0)
    # HICCL_BENCH_RANKS_PER_GPU=k (development): k ranks per GPU, executors
    # sharing it — the N = 8 process/IPC path on a 4-GPU box (no NVLS then)
    share = max(1, int(os.environ.get("HICCL_BENCH_RANKS_PER_GPU", "1")))
    numa_cpus = bind_to_gpu_numa(local // share)
    torch.cuda.set_device(local // share)
    dev = local // share
    p = world
    dtype = args.dtype
    esz = H.ELEMENT_SIZE[dtype]
    S = args.bytes
    d = S // (esz * p)
    S = d * p * esz

    def allgather(obj):
        if pg is None:
            return [obj]
        out = [None] * world
        pg.all_gather_object(out, obj)
        return out

    def max_over_ranks(x: float) -> float:
        if pg is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if pg is not None:
            pg.barrier()

    stream = torch.cuda.Stream(dev)
    sptr = stream.cuda_stream

    def make_comm(kind, form, send_len, recv_len, nvls=False):
        spec = H.CollectiveSpec(H.CollectiveKind(kind), H.Formulation(form), 0, d)
        prog = H.build(spec, p)
        library = ["NVLS"] if nvls else None
        plan = H.lower(prog, H.Machine([p], p, library), ring=1, stripe=1, pipeline=args.pipeline)
        comm = DistCommunicator(plan, rank, world, dev, dtype, ctas=args.ctas, execs_per_device=share,
                                threads=args.threads, copy_mode=args.copy_mode, timeout_s=60.0)
        if nvls:
            where = comm.enable_nvls({"sendbuf": send_len * esz, "recvbuf": recv_len * esz},
                                     allgather)
            send = torch.as_tensor(H.DeviceView(where["sendbuf"], send_len * esz), device=f"cuda:{dev}")
            recv = torch.as_tensor(H.DeviceView(where["recvbuf"], recv_len * esz), device=f"cuda:{dev}")
        else:
            send = torch.empty(send_len * esz, dtype=torch.uint8, device=dev)
            recv = torch.empty(recv_len * esz, dtype=torch.uint8, device=dev)
            comm.register(rank, "sendbuf", send.data_ptr(), send.numel())
            comm.register(rank, "recvbuf", recv.data_ptr(), recv.numel())
        H.device_fill(dev, send.data_ptr(), send_len, dtype, 1234, rank)
        recv.zero_()
        comm.connect(allgather)
        torch.cuda.synchronize(dev)
        return comm, plan, send, recv

    def time_steps(comm, steps, warmup):
        for _ in range(warmup):
            comm.start(sptr)
            comm.wait()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for k in range(steps):
                comm.start(sptr)
                ev[k + 1].record(stream)
        comm.wait()
        torch.cuda.synchronize(dev)
        barrier()
        per = [ev[k].elapsed_time(ev[k + 1]) / 1e3 for k in range(steps)]
        total = ev[0].elapsed_time(ev[steps]) / 1e3
        return total, per

    form = 1 if p > 1 else 0
    # library per the cost model (H.tune_nvls: NVLS wins from p = 4 on)
    nvls = p > 1 and share == 1 and args.nvls != "off" and H.nvls_supported(dev) and (
        args.nvls == "on" or H.tune_nvls(H.CollectiveKind.all_reduce, p, d, dtype)["nvls"])
    nvls = all(allgather(bool(nvls)))
    comm, plan, send, recv = make_comm(7, form, p * d, p * d, nvls=nvls)
    with ClockSampler(dev) as clk:
        total, per = time_steps(comm, args.steps, args.warmup)
    t_total = max_over_ranks(total)
    t_step = t_total / args.steps
    t_kernel = max_over_ranks(statistics.mean(per))
    algbw = S / t_step / 1e9
    busbw = algbw * (2 * (p - 1) / p if p > 1 else 1.0)

    # numerical spot check of the timed result (fp64 sum of every rank's
    # inputs over a slice; tolerance relative to the sum of magnitudes)
    check = {}
    n_chk = min(p * d, 1 << 16)
    acc = np.zeros(n_chk, dtype=np.float64)
    mag = np.zeros(n_chk, dtype=np.float64)
    tmp = torch.empty(n_chk * esz, dtype=torch.uint8, device=dev)
    for r in range(p):
        H.device_fill(dev, tmp.data_ptr(), n_chk, dtype, 1234, r)
        torch.cuda.synchronize(dev)
        x = tmp.cpu().numpy().view(np.float32 if dtype == "f32" else np.uint16)
        x = x.astype(np.float64) if dtype == "f32" else \
            (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        acc += x
        mag += np.abs(x)
    got = recv[: n_chk * esz].cpu().numpy().view(np.float32 if dtype == "f32" else np.uint16)
    got = got.astype(np.float64) if dtype == "f32" else \
        (got.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    rtol = 1e-6 if dtype == "f32" else 1e-2
    err = float(np.max(np.abs(got - acc) / np.maximum(mag, 1e-30)))
    check = {"elements": n_chk, "max_rel_err_vs_sum_abs": err, "rtol": rtol, "ok": err <= rtol}
    digest = float(recv[: 1 << 20].view(torch.float32 if dtype == "f32" else torch.bfloat16)
                   .double().sum().item())
    digests = allgather(digest)
    check["ranks_identical"] = len(set(digests)) == 1

    P = peaks()
    if p == 1:
        achieved = 2 * S / t_kernel / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": P.get("hbm_gbs", 6650.0),
                "unit": "GB/s", "frac": achieved / P.get("hbm_gbs", 6650.0),
                "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                "algorithmic_bytes_per_launch": 2 * S,
                "peak_note": "the measured peak is torch's copy_ (LDG/STG); the executor's TMA "
                             "bulk-copy body can exceed it; HBM3e nominal is 8000 GB/s",
                "frac_of_nominal": achieved / 8000.0}
    else:
        # achieved = busbw = 2S(p-1)/p per GPU per link
        # direction (the point-to-point algorithm's bytes) / kernel time.
        # With NVLS the links actually carry S(1 + 1/p) per direction (the
        # switch reads every member's S and multicasts S back, plus the S/p
        # chunk each GPU sends / draws), reported as link_bytes / link_frac.
        alg_bytes = S * 2 * (p - 1) // p
        achieved = alg_bytes / t_kernel / 1e9
        roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_NOMINAL, "unit": "GB/s",
                "frac": achieved / NVLINK_NOMINAL,
                "frac_of_measured_peer_copy": achieved / NVLINK_MEASURED_PEER,
                "traffic": None,
                "traffic_note": "NVLink bytes one GPU transmits per launch, protocol included, "
                                "from ncu nvltx/nvlrx counters of each executor replayed alone "
                                "(HICCL_PROFILE_SOLO, tools/profile_links.py; profiles/traffic.json); "
                                "NVML's NVLink counters are unsupported on this pool; the multimem "
                                "(NVLS) kernel is captured with ncu --replay-mode application",
                "peak_source": "NVLink 5 nominal 900 GB/s per direction per GPU",
                "algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_bytes_note": "2S(p-1)/p per GPU per link direction (busbw convention)"}
        if nvls:
            link_bytes = S + S // p
            roof["link_bytes_per_launch"] = link_bytes
            roof["link_gbs"] = link_bytes / t_kernel / 1e9
            roof["link_frac"] = roof["link_gbs"] / NVLINK_NOMINAL
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            key = f"all_reduce_p{p}_{S}" + ("_nvls" if nvls else "")
            if key in tj:  # captured on the same schedule (point to point, or NVLS)
                roof["traffic"] = tj[key]
        except Exception:
            pass

    stats = comm.executor.stats()
    result = {
        "metric": "all_reduce_algbw", "value": algbw, "unit": "GB/s", "n_gpus": p,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (counter-hash generator, seed 1234)",
        "config": {"workload": f"all_reduce {'multi (reduce-scatter . all-gather)' if p > 1 else 'single'}"
                               f" p={p} flat {{{p}}}, {S >> 20} MiB per rank",
                   "collective": "all_reduce", "p": p, "hierarchy": [p], "bytes_per_rank": S,
                   "pipeline": args.pipeline, "stripe": 1, "ring": 1, "ctas": stats["ctas"],
                   "threads": stats["threads"], "copy_mode": args.copy_mode,
                   "library": "NVLS (fused multimem.ld_reduce + multimem.st)" if nvls else "p2p",
                   "nvls_items": stats["nvls_items"],
                   "l2": "inputs 1 GiB per rank > 126 MB L2; no flush"},
        "busbw": busbw,
        "roofline": roof,
        "gpu_launches": args.steps,
        "gpu_launches_note": "one persistent executor kernel per step per GPU",
        "clocks": clk.summary(),
        "check": check,
    }

    if not args.no_extras:
        # ---- e2e through the C ABI with host buffers (H2D in, D2H out) ----
        # The all-reduce is elementwise, so the host buffer is streamed in K
        # contiguous pieces, each an all-reduce of its own (one executor per
        # piece bound to its slice of the device buffers): piece k's H2D,
        # piece k-1's collective and piece k-2's D2H overlap on three streams.
        # 16 pieces at N = 1 (46 vs 44 GB/s); 8 when several processes share
        # the host (16 measured slower at N = 4: 12.6 vs 15.0 GB/s)
        K = 16 if (p == 1 and d % 16 == 0) else 8 if d % 8 == 0 else 1
        dk = d // K
        host_in = torch.empty(send.numel(), dtype=torch.uint8, pin_memory=True)
        host_out = torch.empty(recv.numel(), dtype=torch.uint8, pin_memory=True)
        host_in.copy_(send.cpu())
        piece = p * dk * esz
        pieces = []
        for k in range(K):
            spec_k = H.CollectiveSpec(H.CollectiveKind(7), H.Formulation(form), 0, dk)
            plan_k = H.lower(H.build(spec_k, p), H.Machine([p], p), ring=1, stripe=1,
                             pipeline=args.pipeline)
            ck = DistCommunicator(plan_k, rank, world, dev, dtype, ctas=args.ctas, execs_per_device=share,
                                  threads=args.threads, copy_mode=args.copy_mode, timeout_s=60.0)
            if nvls:  # slices of the timed collective's window
                offs = {n: comm.window_offsets[n] + k * piece for n in ("sendbuf", "recvbuf")}
                ck.share_nvls(comm, offs, {"sendbuf": piece, "recvbuf": piece})
            else:
                ck.register(rank, "sendbuf", send.data_ptr() + k * piece, piece)
                ck.register(rank, "recvbuf", recv.data_ptr() + k * piece, piece)
            ck.connect(allgather)
            pieces.append(ck)
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        e2e_steps = max(2, min(args.steps, 5))

        def e2e_once():
            for k, ck in enumerate(pieces):
                lo, hi = k * piece, (k + 1) * piece
                with torch.cuda.stream(s_h2d):
                    send[lo:hi].copy_(host_in[lo:hi], non_blocking=True)
                    ev_in = torch.cuda.Event()
                    ev_in.record(s_h2d)
                stream.wait_event(ev_in)
                ck.start(sptr)
                ev_done = torch.cuda.Event()
                ev_done.record(stream)
                s_d2h.wait_event(ev_done)
                with torch.cuda.stream(s_d2h):
                    host_out[lo:hi].copy_(recv[lo:hi], non_blocking=True)
            s_d2h.synchronize()
            stream.synchronize()

        e2e_once()
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_once()
        torch.cuda.synchronize(dev)
        t_e2e = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
        for ck in pieces:
            ck.wait()
        ok_e2e = bool(torch.equal(host_out[: 1 << 20], recv[: 1 << 20].cpu()))
        for ck in pieces:
            ck.close()
        result["e2e"] = {"value": S / t_e2e / 1e9, "unit": "GB/s",
                         "h2d_bytes_per_step": send.numel(), "d2h_bytes_per_step": recv.numel(),
                         "ms_per_step": t_e2e * 1e3, "pieces": K, "result_matches_device": ok_e2e,
                         "path": "pinned host -> sendbuf (H2D stream), hc_exec_start per piece "
                                 "(compute stream), recvbuf -> pinned host (D2H stream); "
                                 "host wall clock, max over ranks",
                         "host_cpus": len(numa_cpus) if numa_cpus else None}
        del host_in, host_out

        # ---- all-gather (the metric's second collective) ----
        comm.close()
        del send, recv
        torch.cuda.empty_cache()
        ag, _, s2, r2 = make_comm(5, 0, d, p * d)
        ag_total, ag_per = time_steps(ag, args.steps, args.warmup)
        t_ag = max_over_ranks(ag_total) / args.steps
        ag_alg = S / t_ag / 1e9
        result["all_gather"] = {"algbw": ag_alg, "busbw": ag_alg * ((p - 1) / p if p > 1 else 1.0),
                                "ms_per_step": t_ag * 1e3, "unit": "GB/s",
                                "config": f"all_gather single p={p}, recvbuf {S >> 20} MiB per rank"}
        ag.close()
        del s2, r2
        torch.cuda.empty_cache()

        # ---- NCCL on the same box (comparison only; not on our path) ----
        if p > 1:
            try:
                import torch.distributed as dist
                ng = dist.new_group(backend="nccl")
                x = torch.ones(p * d, dtype=torch.float32, device=dev)
                y = torch.empty(p * d, dtype=torch.float32, device=dev)
                for _ in range(args.warmup):
                    dist.all_reduce(x, group=ng)
                torch.cuda.synchronize(dev)
                barrier()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(args.steps):
                    dist.all_reduce(x, group=ng)
                b.record()
                torch.cuda.synchronize(dev)
                t_n = max_over_ranks(a.elapsed_time(b) / 1e3 / args.steps)
                xs = torch.ones(d, dtype=torch.float32, device=dev)
                for _ in range(args.warmup):
                    dist.all_gather_into_tensor(y, xs, group=ng)
                torch.cuda.synchronize(dev)
                barrier()
                a.record()
                for _ in range(args.steps):
                    dist.all_gather_into_tensor(y, xs, group=ng)
                b.record()
                torch.cuda.synchronize(dev)
                t_ng = max_over_ranks(a.elapsed_time(b) / 1e3 / args.steps)
                result["nccl"] = {"all_reduce_algbw": S / t_n / 1e9,
                                  "all_reduce_busbw": S / t_n / 1e9 * 2 * (p - 1) / p,
                                  "all_gather_algbw": S / t_ng / 1e9,
                                  "all_gather_busbw": S / t_ng / 1e9 * (p - 1) / p,
                                  "unit": "GB/s", "version": ".".join(map(str, torch.cuda.nccl.version())),
                                  "env_NVLS": os.environ.get("NCCL_NVLS_ENABLE", "default")}
                del x, y, xs
            except Exception as e:  # comparison only
                result["nccl"] = {"error": str(e)[:200]}
        else:
            result["nccl"] = None

        # ---- CPU baseline: the oracle port on host cores (rank 0, N = 1) ----
        if p == 1 and rank == 0:
            os.sched_setaffinity(0, all_cpus)  # the CPU baseline gets every host core
            import oracle
            from tests import harness
            cores = len(all_cpus)
            sample = 256 << 20
            ds = sample // (esz * p)
            splan, _, _ = harness.make_plan(7, form, p, ds, 0, 0, [p], p, 1, 1, args.pipeline)
            flat = oracle.FlatPlan.from_dicts(splan.world_size, splan.buffers,
                                              splan.transfer_dicts())
            st = harness.initial_state(splan, dtype, 1234)
            oracle.execute(flat, dtype, st, threads=cores)
            reps, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < 3.0 or reps < 3:
                oracle.execute(flat, dtype, st, threads=cores)
                reps += 1
            tc = (time.perf_counter() - t0) / reps
            result["cpu_baseline"] = {"value": ds * p * esz / tc / 1e9, "unit": "GB/s",
                                      "cores": cores, "kind": "port",
                                      "sample": f"{ds * p * esz >> 20} MiB per rank, same plan, "
                                                f"oracle/numeric_exec.c with {cores} threads"}
            result["virtual_c1"] = virtual_c1_leg(args, dev, all_cpus)
    comm.close()
    if rank == 0:
        emit(result)
    barrier()


if __name__ == "__main__":
    main()

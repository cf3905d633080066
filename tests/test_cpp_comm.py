"""hiccl::Comm<T> (include/hiccl/comm.hpp), the paper's C++ user API, built
against libhiccl.so: the header compiles here; on GPUs the paper's
Listing-2 all-reduce runs one process per GPU with a file bootstrap and is
checked bit for bit against the plan's fold order (Comm<float>,
Comm<__nv_bfloat16>, Comm<__half>; on a one-GPU box two processes share the
device)."""
import subprocess
import tempfile
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "comm_demo.cpp"
LIBDIR = ROOT / "paper_2408_05962_b200" / "lib"


def build(out: Path) -> Path:
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", str(SRC), f"-I{ROOT / 'include'}",
           "-I/usr/local/cuda/include", f"-L{LIBDIR}", "-lhiccl", "-L/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_comm_header_compiles(tmp_path):
    assert build(tmp_path / "comm_demo").exists()


@pytest.mark.gpu
@pytest.mark.parametrize("pipeline,dtype", [(1, "f32"), (4, "f32"), (1, "bf16"), (4, "bf16"),
                                            (2, "f16")])
def test_comm_listing2_all_reduce(tmp_path, pipeline, dtype):
    import torch
    exe = build(tmp_path / "comm_demo")
    ngpu = torch.cuda.device_count()
    world = max(2, min(ngpu, 4))  # one GPU: two processes share it
    boot = tempfile.mkdtemp(dir=tmp_path)
    procs = [subprocess.Popen([str(exe), str(r), str(world), str(r % ngpu), "100003", boot,
                               str(pipeline), dtype],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
        assert " 0 mismatches" in o, o
        assert f"{2 if dtype != 'f32' else 4}-byte elements" in o, o


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("pipeline", [1, 2])
def test_comm_listing2_all_reduce_nvls(tmp_path, pipeline):
    # the same composition over Comm::alloc_nvls buffers with library NVLS:
    # every reduce-scatter group and its in-place multicast fuse into one
    # multimem reduce+multicast item per channel
    import torch
    from paper_2408_05962_b200 import hiccl as H
    world = min(torch.cuda.device_count(), 4)
    if world < 2 or not H.nvls_supported(0):
        pytest.skip("needs 2+ GPUs with NVSwitch multicast")
    exe = build(tmp_path / "comm_demo")
    boot = tempfile.mkdtemp(dir=tmp_path)
    procs = [subprocess.Popen([str(exe), str(r), str(world), str(r), "131072", boot, str(pipeline),
                               "nvls"], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
        assert " 0 mismatches" in o and f"{pipeline} nvls items" in o, o

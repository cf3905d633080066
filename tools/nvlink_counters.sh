# NVLink data counters around a 1 GiB all-reduce run (p=4, 20 iterations).
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvl_before.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/sweep.py --sizes 1G --collectives all_reduce --iters 20 --warmup 0 2>&1 | grep '"collective"' > gpurun_out/nvl_run.json
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvl_after.txt 2>&1
head -5 gpurun_out/nvl_before.txt; head -5 gpurun_out/nvl_after.txt; cat gpurun_out/nvl_run.json | head -2

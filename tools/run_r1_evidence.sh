set -u
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x 2>&1 | tail -3
for p in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2952$p tools/sweep.py --sizes 1K,64K,1M,16M,64M,256M,1G --iters 20 --nccl --out gpurun_out/sweep_p$p.jsonl > /dev/null 2>&1
echo "sweep p=$p rc=$?"
done

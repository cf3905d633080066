set -u
mkdir -p gpurun_out
for p in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2958$p tools/sweep.py --sizes 1K,64K,1M,16M,64M,256M,1G --iters 20 --nccl --out gpurun_out/sweep_p$p.jsonl > /dev/null 2>&1
echo "sweep p=$p rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2959$p tools/sweep.py --sizes 1K,64K,1M,16M --collectives all_reduce --formulation single --iters 20 --out gpurun_out/sweep_p${p}_ar_single.jsonl > /dev/null 2>&1
for m in 16 32; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2960$p tools/sweep.py --sizes 64M,256M,1G --collectives broadcast,reduce --formulation single --gpn 1 --ring $p --pipeline $m --iters 10 --out gpurun_out/sweep_p${p}_chain.jsonl > /dev/null 2>&1
done
for m in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2961$p tools/sweep.py --sizes 64M,1G --collectives all_reduce --pipeline $m --iters 10 --out gpurun_out/sweep_p${p}_ar_pipe.jsonl > /dev/null 2>&1
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2962$p tools/sweep.py --sizes 64M,1G --collectives all_reduce,all_gather,reduce_scatter,broadcast --nvls --iters 10 --out gpurun_out/sweep_p${p}_nvls.jsonl > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 2963$p bench.py --gpus $p --steps 10 --warmup 5 2>&1 | grep metric > gpurun_out/bench_p$p.json
echo "p=$p done"
done

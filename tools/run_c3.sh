# BASELINE config C3: all-reduce fp32/bf16 across sizes, GPU "stripes"
# (CTA partitions) x pipeline depth, p=4, vs NCCL.
for dt in f32 bf16; do
for c in 32 74 148; do
for m in 1 4 16; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tools/sweep.py --dtype $dt --sizes 1M,64M,1G --collectives all_reduce --ctas $c --pipeline $m --iters 10 --out gpurun_out/c3_p4.jsonl > /dev/null 2>&1
done; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 tools/sweep.py --dtype $dt --sizes 1K,32K,1M,32M,1G --collectives all_reduce --iters 10 --nccl --out gpurun_out/c3_p4_nccl.jsonl > /dev/null 2>&1
done
echo done

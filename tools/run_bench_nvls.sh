# 4 GPUs: full GPU test suite, bench at p=4 with the NVLS library on / off,
# fused NVLS all-reduce with 256-thread CTAs.
set -u
mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x) > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
for nv in on off; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port $((29710 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 5 --nvls $nv > gpurun_out/bench4_nvls_$nv.log 2>&1
echo "bench nvls=$nv rc=$?"; tail -1 gpurun_out/bench4_nvls_$nv.log | cut -c1-600
done
for th in 256 512; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port $((29810 + RANDOM % 100)) tools/sweep.py --sizes 256M,1G --collectives all_reduce --iters 20 --nvls \
  --threads $th --out gpurun_out/fused_th${th}_p4.jsonl > /dev/null 2>&1
echo "sweep th=$th rc=$?"
done
cat gpurun_out/fused_th*_p4.jsonl | cut -c1-400

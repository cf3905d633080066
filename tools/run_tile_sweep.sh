# 4 GPUs: 1 GiB all-reduce, tile size (HICCL_TILE_VEC) x threads, NVLS fused and p2p.
set -u
mkdir -p gpurun_out
for lib in nvls p2p; do
for th in 256 512; do
for tv in 8 4 2; do
extra=""; [ $lib = nvls ] && extra="--nvls"
HICCL_TILE_VEC=$tv timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 1G --collectives all_reduce --iters 20 $extra \
  --threads $th > gpurun_out/tile_${lib}_${th}_${tv}.log 2>&1
grep '^{' gpurun_out/tile_${lib}_${th}_${tv}.log | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('$lib th=$th tv=$tv', round(r['us'],1), 'busbw', round(r['busbw'],1))"
done; done; done

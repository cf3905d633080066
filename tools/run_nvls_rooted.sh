# 4 GPUs: broadcast / reduce `single` (one multicast / one reduction over
# every rank) lowered to multimem.st / multimem.ld_reduce, against NCCL;
# all-reduce fused NVLS vs point to point across sizes.
set -u
mkdir -p gpurun_out
P=${P:-4}
SIZES=64K,1M,16M,64M,256M,1G
for c in broadcast reduce; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes $SIZES --collectives $c --formulation single \
  --nvls --nccl --iters 20 --out gpurun_out/rooted_nvls_${c}_p$P.jsonl > gpurun_out/rooted_nvls_${c}_p$P.log 2>&1
echo "$c rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes $SIZES --collectives all_reduce \
  --nvls --threads 256 --iters 20 --out gpurun_out/rooted_nvls_ar_p$P.jsonl > gpurun_out/rooted_nvls_ar_p$P.log 2>&1
echo "ar rc=$?"
for f in gpurun_out/rooted_nvls_*_p$P.jsonl; do
python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    r = json.loads(l)
    print(r['impl'], r['collective'], r.get('formulation', ''), r['bytes'], 'us', round(r.get('us', 0), 1),
          'busbw', round(r.get('busbw', 0), 1), 'nvls_items', r.get('nvls_items'), r.get('error', ''))
PY
done

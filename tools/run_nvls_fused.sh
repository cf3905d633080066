# Fused NVLS all-reduce evidence (4 GPUs): tests, hiccl NVLS vs point to
# point vs NCCL (NVLS on and off) at 16 MiB - 1 GiB.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nvls.py -x -q --timeout 300 > gpurun_out/nvls_tests.log 2>&1
echo "nvls tests rc=$?"; tail -3 gpurun_out/nvls_tests.log
P=${P:-4}
run() {  # name, extra args...
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 16M,64M,256M,1G \
    --collectives all_reduce --iters 20 --out gpurun_out/fused_${name}_p$P.jsonl "$@" > gpurun_out/fused_${name}_p$P.log 2>&1
  echo "$name rc=$?"
}
run nvls --nvls
run nvls_m4 --nvls --pipeline 4
HICCL_NO_NVLS_FUSE=1 run nvls_unfused --nvls
run p2p
NCCL_NVLS_ENABLE=1 run nccl_nvls1 --nccl
NCCL_NVLS_ENABLE=0 run nccl_nvls0 --nccl
for f in gpurun_out/fused_*_p$P.jsonl; do
  python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    r = json.loads(l)
    print(sys.argv[1].split('/')[-1], r['impl'], r['collective'], r['bytes'], 'us', round(r['us'], 1),
          'busbw', round(r['busbw'], 1), 'nvls_items', r.get('nvls_items'))
PY
done

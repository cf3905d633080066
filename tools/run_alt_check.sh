# Alternating grid halves per step (HICCL_ALT_HALVES=1) A/B at p=4, plus the
# parity suites with the halves forced on.
set -u
mkdir -p gpurun_out
HICCL_ALT_HALVES=1 timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_multi.py -q -m gpu --timeout 600 -x > gpurun_out/alt_pytest.log 2>&1; echo "pytest(alt) rc=$?"; tail -1 gpurun_out/alt_pytest.log
rm -f gpurun_out/alt_*.jsonl
for a in 1 0; do
  O=gpurun_out/alt_$a.jsonl
  for c in reduce broadcast; do for m in 8 16 32; do
    HICCL_ALT_HALVES=$a timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 16M,64M,256M,1G --collectives $c --formulation single --gpn 1 --ring 4 --pipeline $m --iters 10 --out $O > /dev/null 2>&1
  done; done
  HICCL_ALT_HALVES=$a timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 64M,1G --collectives all_reduce --pipeline 4 --iters 10 --out $O > /dev/null 2>&1
  HICCL_ALT_HALVES=$a timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 64M,1G --collectives all_reduce --iters 10 --out $O > /dev/null 2>&1
  echo "alt=$a done"
done
python - <<'PY'
import json
rows = {}
for a in ("1", "0"):
    for l in open(f"gpurun_out/alt_{a}.jsonl"):
        r = json.loads(l)
        rows.setdefault((r["collective"], r["pipeline"], r["bytes"]), {})[a] = r["us"]
for k in sorted(rows):
    v = rows[k]
    print(k[0], "m", k[1], k[2] >> 20, "MiB", "alt", round(v.get("1", 0), 1), "base", round(v.get("0", 0), 1))
PY

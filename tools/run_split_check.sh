# Warp-specialized step loop A/B (HICCL_NO_SPLIT_SYNC=1 = the old single
# loop) at p=4: GPU tests, main collectives, chains, pipelined all-reduce.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/sc_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/sc_pytest.log
rm -f gpurun_out/sc_*.jsonl
for mode in split nosplit; do
  env=""; [ $mode = nosplit ] && env="HICCL_NO_SPLIT_SYNC=1"
  env $env timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 1M,16M,64M,1G --collectives all_reduce,all_gather --iters 20 --out gpurun_out/sc_${mode}.jsonl > /dev/null 2>&1
  env $env timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 1M,16M,64M,1G --collectives all_reduce --pipeline 4 --iters 20 --out gpurun_out/sc_${mode}.jsonl > /dev/null 2>&1
  for c in broadcast reduce; do for m in 8 16; do
    env $env timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 16M,64M,256M,1G --collectives $c --formulation single --gpn 1 --ring 4 --pipeline $m --iters 10 --out gpurun_out/sc_${mode}.jsonl > /dev/null 2>&1
  done; done
  echo "$mode done"
done
python - <<'PY'
import json
rows = {}
for mode in ("split", "nosplit"):
    for l in open(f"gpurun_out/sc_{mode}.jsonl"):
        r = json.loads(l)
        rows.setdefault((r["collective"], r["pipeline"], r["bytes"]), {})[mode] = r["us"]
for k in sorted(rows):
    v = rows[k]
    print(k[0], "m", k[1], k[2] >> 20, "MiB", "split", round(v.get("split", 0), 1), "nosplit", round(v.get("nosplit", 0), 1))
PY

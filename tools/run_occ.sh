# Two 256-thread CTAs per SM against one 512-thread CTA: chains and 1 GiB collectives, p=4.
set -u
O=gpurun_out/occ.jsonl; rm -f $O
for cfg in "512 148" "256 296" "256 148"; do
  set -- $cfg; th=$1; g=$2
  for c in broadcast reduce; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 16M,64M,256M,1G --collectives $c --formulation single --gpn 1 --ring 4 --pipeline 16 --iters 10 --threads $th --ctas $g --out $O > /dev/null 2>&1
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 16M,64M,1G --collectives all_reduce,all_gather,reduce_scatter --iters 10 --threads $th --ctas $g --out $O > /dev/null 2>&1
  echo "$cfg done"
done
python - <<'PY'
import json
rows = {}
for l in open("gpurun_out/occ.jsonl"):
    r = json.loads(l)
    rows.setdefault((r["collective"], r["bytes"]), []).append((r["ctas"], round(r["us"], 1)))
for k in sorted(rows):
    print(k[0], k[1] >> 20, "MiB", rows[k])
PY

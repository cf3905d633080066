# Deferred accumulator init + placement (push schedules): GPU tests, chains,
# main collectives and the {2,4} configuration at p=4.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pc_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pc_pytest.log
O=gpurun_out/pc.jsonl; rm -f $O
for c in reduce broadcast; do for m in 8 16 32; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 16M,64M,256M,1G --collectives $c --formulation single --gpn 1 --ring 4 --pipeline $m --iters 10 --out $O > /dev/null 2>&1
done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 1M,64M,1G --collectives all_reduce,all_gather,reduce_scatter --iters 10 --out $O > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --ranks-per-gpu 2 --sizes 64M --collectives all_reduce --hierarchy 2,4 --gpn 4 --stripe 4 --ring 2 --iters 10 --out $O > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 1G --collectives reduce_scatter --hierarchy 2,2 --gpn 2 --stripe 2 --iters 10 --out $O > /dev/null 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/pc.jsonl"):
    r = json.loads(l)
    if "error" in r: print("ERR", r); continue
    print(r["collective"], r["hierarchy"], "m", r["pipeline"], r["bytes"] >> 20, "MiB", round(r["us"], 1), "us busbw", round(r["busbw"], 1))
PY

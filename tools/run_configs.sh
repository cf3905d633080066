# BASELINE.json configurations C1, C4, C5 at full size: 8 logical ranks on
# 4 GPUs (2 per GPU, virtual hierarchies) and the 2-level {2,2} on 4 GPUs.
set -u
mkdir -p gpurun_out
O=gpurun_out/configs.jsonl; rm -f $O
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) tools/sweep.py --iters 10 --warmup 3 --out $O "$@" > /dev/null 2>&1; echo "rc=$? $*"; }
# C1: all-reduce 64 MiB/rank, p=8 on {2,4} g=4, tree / ring 2, s 1 / 4, m 1 / 4
for s in 1 4; do for n in 1 2; do for m in 1 4; do
  run --ranks-per-gpu 2 --sizes 64M --collectives all_reduce --hierarchy 2,4 --gpn 4 --stripe $s --ring $n --pipeline $m
done; done; done
# C4: all-gather / reduce-scatter 1 GiB on {2,2,2}: g=8, and g=2 with s=2
for c in all_gather reduce_scatter; do
  run --ranks-per-gpu 2 --sizes 1G --collectives $c --hierarchy 2,2,2 --gpn 8
  run --ranks-per-gpu 2 --sizes 1G --collectives $c --hierarchy 2,2,2 --gpn 2 --stripe 2
  run --sizes 1G --collectives $c --hierarchy 2,2 --gpn 2 --stripe 2
  run --sizes 1G --collectives $c
done
# C5: all-to-all 8 MiB - 1 GiB per rank, {8} and {2,4} g=4 ring 2 (virtual p=8), flat {4}
run --ranks-per-gpu 2 --sizes 8M,64M,1G --collectives all_to_all
run --ranks-per-gpu 2 --sizes 8M,64M,1G --collectives all_to_all --hierarchy 2,4 --gpn 4 --ring 2
run --sizes 8M,64M,1G --collectives all_to_all --nccl
python - <<'PY'
import json
for l in open("gpurun_out/configs.jsonl"):
    r = json.loads(l)
    if "error" in r:
        print("ERR", r); continue
    print(r["impl"], r["collective"], r["p"], r.get("hierarchy"), "g", r.get("g"), "s", r.get("stripe"), "n", r.get("ring"),
          "m", r.get("pipeline"), r["bytes"] >> 20, "MiB", round(r["us"], 1), "us algbw", round(r["algbw"], 1))
PY

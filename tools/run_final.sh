# Final round-1 check on 4 GPUs: smoke, GPU tests, default choices for the
# rooted collectives, and bench at N = 1, 2, 4 (reference arm first).
set -u
mkdir -p gpurun_out
O=gpurun_out/final_rooted_p4.jsonl; rm -f $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 tools/sweep.py --sizes 1M,16M,64M,256M,1G --collectives broadcast,reduce --auto --nvls --nccl --iters 20 --out $O > /dev/null 2>&1; echo "rooted rc=$?"
python - <<'PY'
import json
rows = {}
for l in open("gpurun_out/final_rooted_p4.jsonl"):
    r = json.loads(l)
    rows.setdefault((r["collective"], r["bytes"]), {})[r["impl"]] = r
for (c, b), v in sorted(rows.items()):
    h, n = v.get("hiccl", {}), v.get("nccl", {})
    print(c, b >> 20, "MiB hiccl", round(h.get("us", 0), 1), h.get("formulation"), "m", h.get("pipeline"),
          "nvls" if h.get("nvls") else h.get("copy_mode"), "| nccl", round(n.get("us", 0), 1) if n else "-")
PY
bash tools/run_round_end.sh

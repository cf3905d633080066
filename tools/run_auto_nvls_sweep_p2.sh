# p=4: what a user gets by default with buffers in an NVLS window — every
# collective with the cost model's choice (tune_nvls: formulation, ring,
# pipeline, copy mode, NVLS or point to point) against NCCL.
set -u
O=gpurun_out/auto_nvls_all_p2.jsonl; rm -f $O
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691 tools/sweep.py --sizes 1K,64K,1M,16M,64M,256M,1G --collectives all_reduce,all_gather,reduce_scatter,all_to_all,broadcast,reduce,scatter,gather --auto --nvls --nccl --iters 20 --out $O > gpurun_out/auto_nvls_all_p2.log 2>&1
echo "rc=$?"
python - <<'PY'
import json
rows = {}
for l in open("gpurun_out/auto_nvls_all_p2.jsonl"):
    r = json.loads(l)
    rows.setdefault((r["collective"], r["bytes"]), {})[r["impl"]] = r
for (c, b), v in sorted(rows.items()):
    h, n = v.get("hiccl", {}), v.get("nccl", {})
    print(c, b, "hiccl", round(h.get("us", 0), 1), h.get("formulation"), "m", h.get("pipeline"), h.get("copy_mode"),
          "nvls" if h.get("nvls") else "p2p", "| nccl", round(n.get("us", 0), 1) if n else "-")
PY

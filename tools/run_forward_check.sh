# Copy forwarding (reduce-scatter into __tmp + gather -> one fold stored at
# the root): GPU tests, reduce multi / single with and without NVLS vs NCCL, p=4.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/fw_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fw_pytest.log
O=gpurun_out/fw.jsonl; rm -f $O
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 1M,16M,64M,256M,1G --collectives reduce --iters 20 --out $O "$@" > /dev/null 2>&1; echo "rc=$? $*"; }
run --formulation multi --nvls
run --formulation multi --nccl
run --formulation single --nvls
python - <<'PY'
import json
for l in open("gpurun_out/fw.jsonl"):
    r = json.loads(l)
    print(r["impl"], r.get("formulation", ""), "nvls" if r.get("nvls") else "", r["bytes"] >> 20, "MiB", round(r["us"], 1), "us")
PY

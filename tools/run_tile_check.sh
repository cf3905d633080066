# After a layout change: GPU tests (4 GPUs), chain traces, and a p=4 sweep
# of the main collectives against the committed round-1 numbers.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/tc_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/tc_pytest.log
bash tools/run_chain_trace64.sh > gpurun_out/tc_chain.log 2>&1; grep -E "^(reduce|broadcast)" gpurun_out/tc_chain.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29677 tools/sweep.py --sizes 1M,16M,64M,256M,1G --collectives all_reduce,all_gather,reduce_scatter,all_to_all --iters 20 --out gpurun_out/tc_sweep_p4.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
for c in broadcast reduce; do for m in 8 16 32; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29680 + m)) tools/sweep.py --sizes 16M,64M,256M,1G --collectives $c --formulation single --gpn 1 --ring 4 --pipeline $m --iters 10 --out gpurun_out/tc_chain_p4.jsonl > /dev/null 2>&1
done; done
python - <<'PY'
import json
for f in ("gpurun_out/tc_sweep_p4.jsonl", "gpurun_out/tc_chain_p4.jsonl"):
    for l in open(f):
        r = json.loads(l)
        print(r["collective"], r["bytes"] >> 20, "MiB m", r["pipeline"], "us", round(r["us"], 1), "busbw", round(r["busbw"], 1))
PY

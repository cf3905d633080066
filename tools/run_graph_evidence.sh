# Graph-replayed sweeps (device-side latency, no host launch cost) at p=4 and p=2:
# tagged lines (both formulations), push, NCCL, and the cost model's auto choice.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
SZ=1K,16K,64K,256K,1M,4M,16M,64M
for np in 4 2; do
  run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $1 tools/sweep.py --iters 50 --graph "${@:2}" > /dev/null 2>&1; }
  run 29581 --sizes $SZ --collectives all_reduce,broadcast,reduce --formulation single --copy-mode ll --out gpurun_out/ll_graph_p${np}_single.jsonl
  run 29582 --sizes $SZ --collectives all_reduce,broadcast,reduce --formulation multi --copy-mode ll --out gpurun_out/ll_graph_p${np}_multi.jsonl
  run 29583 --sizes $SZ --collectives all_gather,reduce_scatter,all_to_all,scatter,gather --copy-mode ll --out gpurun_out/ll_graph_p${np}_rest.jsonl
  run 29584 --sizes $SZ --copy-mode push --nccl --out gpurun_out/push_nccl_graph_p${np}.jsonl
  run 29585 --sizes $SZ --auto --out gpurun_out/auto_graph_p${np}.jsonl
done
ls -la gpurun_out/*.jsonl

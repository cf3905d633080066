timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 tools/sweep.py --dtype bf16 --sizes 64M,1G --collectives all_reduce,reduce_scatter,all_gather --iters 10 --nccl --out gpurun_out/sweep_p4_bf16.jsonl 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('bf16', r['impl'], r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))"

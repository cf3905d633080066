timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/sweep.py --sizes 1K,16K,256K,1M,4M,16M,64M,256M,1G --collectives all_reduce,all_gather --iters 20 --nccl --out gpurun_out/sweep_p4.jsonl 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['impl'], r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))"

./tools/nvlinkbench_p
for nv in 0 1; do
NCCL_NVLS_ENABLE=$nv timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2951$nv tools/sweep.py --sizes 64M,1G --collectives all_reduce,all_gather --iters 10 --nccl 2>&1 | grep '"nccl"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('NVLS=$nv', r['impl'], r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))"
done
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 tools/sweep.py --sizes 1G --collectives all_reduce --iters 3 --nccl 2>&1 | grep -iE "nvls|algo|protocol" | head -20

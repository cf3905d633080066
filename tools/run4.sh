timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 2>&1 | tail -2
for mode in pull push; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py --sizes 1G --collectives all_reduce,all_gather,reduce_scatter,all_to_all --copy-mode $mode --iters 10 --nccl 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['impl'], r.get('copy_mode',''), r['collective'], r['bytes'], 'us', round(r['us']), 'busbw', round(r['busbw']))"
done

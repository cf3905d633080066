for m in 1 2 4 8 16; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29563 tools/sweep.py --sizes 256M,1G --collectives all_reduce --nvls --pipeline $m --iters 8 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('NVLS m=$m', r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1), 'nvls_items', r['nvls_items'], 'steps', r['steps'])"
done
for m in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29564 tools/sweep.py --sizes 256M,1G --collectives all_reduce --pipeline $m --iters 8 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('P2P m=$m', r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))"
done

timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 tools/sweep.py --sizes 1K,1M,16M,64M,1G --collectives all_reduce,all_gather --iters 10 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))"
for m in 8 16 32 64; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 tools/sweep.py --sizes 64M,1G --collectives broadcast,reduce --formulation single --gpn 1 --ring 4 --pipeline $m --iters 8 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('chain m=$m', r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))"
done

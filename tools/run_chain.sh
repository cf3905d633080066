for m in 8 16 32 64; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/sweep.py --sizes 64M,1G --collectives broadcast,reduce --formulation single --gpn 1 --ring 4 --pipeline $m --iters 10 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('m=$m', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1), r.get('steps'), r.get('error',''))"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/sweep.py --sizes 1K,64K,1M,4M,16M --collectives all_reduce --formulation single --iters 20 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('AR single', r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1))"

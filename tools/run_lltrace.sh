timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "ll" 2>&1 | tail -2
for np in 4 2; do
for f in multi single; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29571 tools/sweep.py --sizes 1K,16K,64K,256K,1M,4M --collectives all_reduce,broadcast,reduce --formulation $f --copy-mode ll --iters 50 --graph 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l)
    print('p=$np $f', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'ctas', r['ctas'])"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29572 tools/sweep.py --sizes 1K,16K,64K,256K,1M,4M --collectives all_gather,reduce_scatter,all_to_all --copy-mode ll --iters 50 --graph 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l)
    print('p=$np', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'ctas', r['ctas'])"
done

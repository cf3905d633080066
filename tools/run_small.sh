timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/sweep.py --sizes 1K,256K,4M,16M,64M,1G --collectives all_reduce,all_gather --iters 20 --trace 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['impl'], r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1), json.dumps(r.get('trace')))"

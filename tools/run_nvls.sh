timeout 600 python -m pytest tests/test_gpu_nvls.py -x -q --timeout 200 2>&1 | tail -15
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/sweep.py --sizes 1M,16M,64M,256M,1G --collectives all_reduce,all_gather,reduce_scatter,broadcast --nvls --iters 10 2>&1 | grep -E '"collective"|Error|error' | python -c "
import json,sys
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print('NVLS', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1), 'nvls_items', r.get('nvls_items'), r.get('error',''))"

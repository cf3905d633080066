timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/sweep.py --sizes 1G --collectives broadcast --formulation single --gpn 1 --ring 4 --pipeline 16 --iters 5 --trace 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['collective'], r['bytes'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))
    for rk, t in enumerate(r['trace']):
        st=[round(x,1) if x else None for x in t['steps_us']]
        print(' rank', rk, 'entry', t['entry_barrier_us'], 'steps', st, 'last', t['last_cta_us'], 'exit', t['exit_us'])"

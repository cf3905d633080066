for cfg in "--ctas 148 --threads 512" "--ctas 296 --threads 256" "--ctas 148 --threads 256"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 tools/sweep.py --sizes 1G --collectives all_reduce,reduce_scatter,all_gather --nvls --iters 5 --trace $cfg 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('$cfg', r['collective'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1))
    for rk, t in enumerate(r['trace'][:2]):
        st=[round(x,1) if x else None for x in t['steps_us']]
        print('   rank', rk, 'entry', t['entry_barrier_us'], 'steps', st, 'last', t['last_cta_us'], 'exit', t['exit_us'])"
done

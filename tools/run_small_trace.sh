for f in multi single; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-4} --master-addr 127.0.0.1 --master-port 29591 tools/sweep.py --sizes 1K,1M --collectives all_reduce --formulation $f --iters 20 --trace 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('$f', r['bytes'], 'us', round(r['us'],1), 'ctas', r['ctas'])
    for rk, t in enumerate(r['trace'][:2]):
        print('   rank', rk, 'entry', t['entry_barrier_us'], 'steps', t['steps_us'], 'last', t['last_cta_us'], 'exit', t['exit_us'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-4} --master-addr 127.0.0.1 --master-port 29592 tools/sweep.py --sizes 1K --collectives all_gather --iters 20 --trace 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('AG', r['bytes'], 'us', round(r['us'],1), 'ctas', r['ctas'])
    for rk, t in enumerate(r['trace'][:2]):
        print('   rank', rk, 'entry', t['entry_barrier_us'], 'steps', t['steps_us'], 'last', t['last_cta_us'], 'exit', t['exit_us'])"

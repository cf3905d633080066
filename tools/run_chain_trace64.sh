# p=4 chain reduce / broadcast at 64 MiB with the device timeline (CTA 0's
# step publishes per rank), m = 8 and 16.
for c in reduce broadcast; do
for m in 8 16; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/sweep.py --sizes 64M --collectives $c --formulation single --gpn 1 --ring 4 --pipeline $m --iters 10 --trace 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['collective'], r['bytes'], 'm', r['pipeline'], 'us', round(r['us'],1), 'busbw', round(r['busbw'],1), 'ctas', r['ctas'])
    for rk, t in enumerate(r['trace']):
        st=[round(x,1) if x else None for x in t['steps_us']]
        print(' rank', rk, 'entry', t['entry_barrier_us'], 'steps', st, 'last', t['last_cta_us'], 'exit', t['exit_us'])"
done; done

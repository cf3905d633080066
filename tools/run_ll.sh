# Tagged-line (ll) mode: parity on 2/4 GPUs, then small-message latency vs push at p=4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "ll" 2>&1 | tail -15
for mode in ll push; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-4} --master-addr 127.0.0.1 --master-port 29561 tools/sweep.py --sizes 1K,16K,64K,256K,1M,4M,16M --collectives all_reduce,all_gather,reduce_scatter,broadcast,all_to_all --copy-mode $mode --iters 20 --trace 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); t=r.get('trace',[{}])[0] if r.get('trace') else {}
    print('$mode', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1), 'ctas', r.get('ctas'), 'entry', t.get('entry_barrier_us'), 'steps', t.get('steps_us'), 'last', t.get('last_cta_us'), r.get('error',''))"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-4} --master-addr 127.0.0.1 --master-port 29562 tools/sweep.py --sizes 1K,16K,64K,256K,1M,4M,16M --collectives all_reduce --formulation single --copy-mode ll --iters 20 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('ll-single', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1), r.get('error',''))"

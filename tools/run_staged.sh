# Staged copy mode: parity first, then push vs staged at p=4.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "staged" 2>&1 | tail -5
for mode in push staged; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/sweep.py --sizes 1M,16M,256M,1G --collectives all_reduce,reduce_scatter,reduce --copy-mode $mode --iters 10 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('$mode', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1), r.get('error',''))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tools/sweep.py --sizes 64M,1G --collectives reduce --formulation single --gpn 1 --ring 4 --pipeline 32 --copy-mode $mode --iters 10 2>&1 | grep '"collective"' | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('$mode chain', r['collective'], r['bytes'], 'us', round(r.get('us',0),1), 'busbw', round(r.get('busbw',0),1), r.get('error',''))"
done

set -x
python tools/probe.py 2>&1 | tail -7
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 2>&1 | tail -2
for args in "" "--copy-mode push" "--pipeline 4" "--pipeline 4 --copy-mode push"; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-extras $args 2>&1 | grep metric | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$args', 'algbw', round(r['value'],1), 'busbw', round(r['busbw'],1), 'ms', round(r['ms_per_step'],3), r['check']['ok'], r['clocks'])"
done

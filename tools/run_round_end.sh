# What the driver runs at round end, on this box's GPUs: smoke(), the GPU
# tests, bench.py (reference arm first) at N = 1 and, with more GPUs, N > 1.
set -u
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/re_smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/re_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/re_pytest.log
python bench.py --impl reference > gpurun_out/re_ref1.log 2>&1; echo "ref1 rc=$?"; tail -1 gpurun_out/re_ref1.log | cut -c1-300
python bench.py > gpurun_out/re_bench1.log 2>&1; echo "bench1 rc=$?"; tail -1 gpurun_out/re_bench1.log | cut -c1-400
for n in 2 4 8; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --impl reference --gpus $n > gpurun_out/re_ref$n.log 2>&1; echo "ref$n rc=$?"; grep '^{' gpurun_out/re_ref$n.log | cut -c1-300
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29510 + n)) bench.py --gpus $n > gpurun_out/re_bench$n.log 2>&1; echo "bench$n rc=$?"; grep '^{' gpurun_out/re_bench$n.log | cut -c1-400
done

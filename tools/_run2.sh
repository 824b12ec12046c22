mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pt.log | grep -v "^$" | tail -8
for D in 7 5; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --degree $D > gpurun_out/b1.log 2>&1; echo "N=$D rc=$? $(grep -o '"value": [0-9.]*\|"ms_per_iteration": [0-9.]*\|"k1_ms": [0-9.]*\|"k2_ms": [0-9.]*\|"frac": [0-9.]*' gpurun_out/b1.log | tr '\n' ' ')"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py > gpurun_out/dc2.log 2>&1; echo dc=$?; tail -2 gpurun_out/dc2.log
for E in "32 32 32" "64 64 64"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --elements $E > gpurun_out/b2.log 2>&1
  echo "$E rc=$? $(grep -o '"value": [0-9.]*\|"ms_per_iteration": [0-9.]*\|"k1_ms": [0-9.]*\|"rest_of_iteration_ms": [0-9.]*' gpurun_out/b2.log | tr '\n' ' ')"
done

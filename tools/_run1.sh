for G in 0 1; do
if [ $G = 1 ]; then export SBX_K2_NOGATHER=1; fi
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --iters 20 > gpurun_out/b1.log 2>&1; echo "nogather=$G rc=$? $(grep -o '"ms_per_iteration": [0-9.]*\|"k1_ms": [0-9.]*\|"k2_ms": [0-9.]*' gpurun_out/b1.log | tr '\n' ' ')"
done

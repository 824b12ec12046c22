#!/bin/bash
# Strong-scaling / size / degree sweep (SURVEY §8(d) C3-C5 on the GPUs of one
# box).  Usage (from the repo root, on the GPU box):  bash tools/sweep.sh NGPUS
# Appends one bench.py JSON line per run to gpurun_out/sweep.jsonl.
set -u
G=${1:-4}
OUT=gpurun_out/sweep.jsonl
mkdir -p gpurun_out
run() {  # gpus degree ex ey ez
  local g=$1 d=$2; shift 2
  if [ "$g" = 1 ]; then
    timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ax-microbench \
      --degree $d --elements "$@" > gpurun_out/sw.log 2>&1
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $g --steps 3 --warmup 3 \
      --no-cpu-baseline --no-ax-microbench --degree $d --elements "$@" > gpurun_out/sw.log 2>&1
  fi
  local rc=$?
  local l=$(grep '^{"metric"' gpurun_out/sw.log | tail -1)
  if [ -n "$l" ]; then echo "$l" >> $OUT; else echo "{\"failed\": \"g=$g d=$d e=$*\", \"rc\": $rc}" >> $OUT; fi
  echo "g=$g N=$d E=$* rc=$rc"
}
for E in "16 16 16" "20 20 20" "24 24 24" "32 32 32" "48 48 48" "64 64 64"; do
  for g in 1 2 4; do
    [ $g -le $G ] && run $g 7 $E
  done
done
for d in 5 9; do
  for g in 1 2 4; do
    [ $g -le $G ] && run $g $d 64 64 64
  done
done

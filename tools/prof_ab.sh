for i in 1 2; do
  for p in mode0 none full; do
    export TSG_BENCH_PROF=$p
    python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.log 2>&1
    echo "prof=$p steps100 $(grep -o '"value": [0-9.]*' gpurun_out/bg.log | head -1)"
  done
done
export TSG_BENCH_PROF=mode0
python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.log 2>&1
echo "prof=mode0 default $(grep -o '"value": [0-9.]*' gpurun_out/bg.log | head -1)"

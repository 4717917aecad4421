for i in 1 2 3; do
  for g in 0 1; do
    if [ $g = 1 ]; then export TSG_NO_GRAPH=1; else unset TSG_NO_GRAPH; fi
    python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.log 2>&1
    echo "nograph=$g $(grep -o '"value": [0-9.]*' gpurun_out/bg.log | head -1)"
  done
done

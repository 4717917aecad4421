for i in 1 2 3; do
  for c in 0 1; do
    export TSG_TAIL_LDCS=$c
    python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.log 2>&1
    echo "ldcs=$c $(grep -o '"value": [0-9.]*' gpurun_out/bg.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/bg.log)"
  done
done

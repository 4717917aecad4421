for i in 1 2; do
  for c in 0 100 64 32; do
    if [ $c = 0 ]; then unset TSG_TAIL_CTAS; else export TSG_TAIL_CTAS=$c; fi
    python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.log 2>&1
    echo "tail=$c $(grep -o '"value": [0-9.]*' gpurun_out/bg.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/bg.log)"
  done
done

for i in 1 2; do
  for c in 0 296 264 248; do
    if [ $c = 0 ]; then unset TSG_M0_CTAS; else export TSG_M0_CTAS=$c; fi
    python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.log 2>&1
    echo "m0=$c $(grep -o '"value": [0-9.]*' gpurun_out/bg.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/bg.log)"
  done
done

for f in 1 8 16 28; do
  export TSG_PROJ_FREE_SMS=$f
  python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_c3.log 2>&1
  echo "free=$f $(grep -o '"value": [0-9.]*' gpurun_out/b_c3.log | head -1) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/b_c3.log)"
done

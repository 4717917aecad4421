for c in 0 272 256 232; do
  if [ $c = 0 ]; then unset TSG_M0_CTAS; else export TSG_M0_CTAS=$c; fi
  python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bs.log 2>&1
  tail -1 gpurun_out/bs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})"
done

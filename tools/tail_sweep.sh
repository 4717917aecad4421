run() {
  python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bs.log 2>&1
  tail -1 gpurun_out/bs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('m0=${TSG_M0_CTAS:-def} tail=${TSG_TAIL_CTAS:-def}', round(d['value']), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})"
}
run
export TSG_M0_CTAS=264; export TSG_TAIL_CTAS=24; run
export TSG_M0_CTAS=264; export TSG_TAIL_CTAS=16; run
export TSG_M0_CTAS=248; export TSG_TAIL_CTAS=32; run
export TSG_M0_CTAS=232; export TSG_TAIL_CTAS=48; run
export TSG_M0_CTAS=280; export TSG_TAIL_CTAS=48; run

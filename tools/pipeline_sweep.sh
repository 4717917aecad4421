#!/bin/bash
run() { echo "== $*"; env "$@" python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['roofline']['frac'],3), {k:round(v*1e3,1) for k,v in d['phases_ms'].items()}, round(d['events_pass_ms_per_step']*1e3,1))
"; }
run TSG_TAIL_CTAS=148
run TSG_TAIL_CTAS=8
run TSG_TAIL_CTAS=16 TSG_COLS0_FREE_SMS=16
run TSG_TAIL_CTAS=8 TSG_ISVD_CTA=2
run TSG_TAIL_CTAS=16 TSG_COLS0_FREE_SMS=16 TSG_ISVD_CTA=2
run TSG_TAIL_CTAS=24 TSG_COLS0_FREE_SMS=24
run TSG_PROJ0_COLS=0 TSG_PROJ0_FMA=0
run TSG_PROJ0_COLS=0 TSG_PROJ0_FMA=0 TSG_ISVD_CTA=0

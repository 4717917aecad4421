#!/bin/bash
# Prints value / roofline frac / phases / events-pass period of bench.py runs: bench_brief.sh [ENV=..] -- [bench args]
envs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
echo "== ${envs[*]} $*"
env "${envs[@]}" python bench.py "$@" 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print(round(d['value']), 'us/slice', round(d['ms_per_step']*1e3,1), 'frac', r.get('frac') and round(r['frac'],3), {k:round(v*1e3,1) for k,v in d.get('phases_ms',{}).items()}, 'evpass', d.get('events_pass_ms_per_step') and round(d['events_pass_ms_per_step']*1e3,1), 'e2e', d['e2e'] and round(d['e2e']['value']), 'steps', d['steps'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    elif 'Error' in l or 'error' in l: print(l.strip())
"

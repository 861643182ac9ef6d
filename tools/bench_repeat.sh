#!/bin/bash
# Run the default bench line N times (run-to-run variance); prints one summary JSON per run.
N=${1:-3}; shift
for i in $(seq 1 $N); do
  timeout 300 python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1 | RUN=$i python -c "
import json, os, sys
d = json.loads(sys.stdin.read())
print(json.dumps({'run': int(os.environ['RUN']), 'value': d['value'], 'ms_per_step': d['ms_per_step'],
                  'frac': d['roofline']['frac'], 'e2e': d['e2e']['value'], 'clocks': d['clocks']}))"
done

#!/bin/bash
# A/B of the bins-per-step batch size (full waves of the persistent CTA pairs vs a ragged last wave)
run() { # config bins steps
  python bench.py --config $1 --bins-per-step $2 --steps $3 --warmup 3 --no-parity --no-cpu-baseline 2>/dev/null \
   | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('$1', $2, d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
}
for b in 2048 2072 2035 2048 2072; do run c5 $b 5; done
for b in 4096 4144 4096 4144; do run c2 $b 10; done
for b in 1024 1036 1024 1036; do run c4 $b 5; done

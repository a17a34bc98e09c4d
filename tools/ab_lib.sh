#!/bin/bash
# Same-box A/B of two builds of libcider (paper_2605_26580_b200/_lib vs $1): alternating c5 / c2 bench runs
ALT=$1; shift
run() { # tag config libdir
  CIDER_LIB_DIR=$3 timeout 300 python bench.py --config $2 --steps 5 --warmup 3 --no-parity --no-cpu-baseline 2>/dev/null \
   | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); k=d['roofline']['kernels']; print('$1', '$2', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], {n:k[n]['ms'] for n in ('embed','gemm_logits','mlp_agg') if n in k})"
}
for i in 1 2 3; do
  for c in "$@"; do run new $c $PWD/paper_2605_26580_b200/_lib; run base $c $ALT; done
done

#!/bin/bash
# co-run bench per library variant (scripts/variants.py build ...): bash scripts/gpu_variants_bench.sh tag1 tag2 ...
cd "$(dirname "$0")/.."
for t in "$@"; do
  echo "== $t"
  SEMIPD_LIB=$PWD/paper_2504_19867_b200/libsemipd_v_$t.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],3), d['config']['split'], 'dec TB/s', round(d['roofline_decode']['achieved']), 'pre TF/s', round(d['roofline_prefill']['achieved']), 'step', round(d['roofline_step']['frac'],3), d['corun_streams'], [(s['x'], round(s['tokens_per_s'])) for s in d['sweep']])"
done

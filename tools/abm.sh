#!/usr/bin/env bash
# multi-variant interleaved A/B: /tmp/abm.sh "<bench args>" reps lib1 lib2 ...
ARGS="$1"; REPS="$2"; shift 2
for r in $(seq 1 $REPS); do
  for L in "$@"; do
    v=$(BBK_LIB=$L python bench.py $ARGS --no-cpu-baseline --no-e2e --no-sweep --no-games --no-reference-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'{d[\"value\"]/1e6:.2f}M frac={d[\"roofline\"][\"frac\"]:.3f}')")
    echo "$ARGS $L: $v"
  done
done

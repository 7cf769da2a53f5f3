#!/usr/bin/env bash
# A/B: run the same bench with two library builds, interleaved, in one GPU session.
# usage: tools/ab.sh "<bench args>" ab/libA.so ab/libB.so [reps]
ARGS="$1"; A="$2"; B="$3"; REPS="${4:-2}"
for r in $(seq 1 $REPS); do
  for L in "$A" "$B"; do
    v=$(BBK_LIB=$L python bench.py $ARGS --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'{d[\"value\"]/1e6:.2f}M frac={d[\"roofline\"][\"frac\"]:.3f} kern={d[\"roofline\"][\"kernel_ms\"]:.3f}ms')")
    echo "$L: $v"
  done
done

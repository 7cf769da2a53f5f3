#!/usr/bin/env bash
# ncu --set full capture of one mid-episode step-kernel launch for the given games (default go_9x9 go_19x19)
OUT=gpurun_out; mkdir -p $OUT
for spec in ${@:-go_9x9:60 go_19x19:250}; do
  g=${spec%%:*}; w=${spec##*:}
  python bench.py --game $g --steps 2 --warmup $w --no-cpu-baseline --no-e2e --no-sweep > $OUT/plain_$g.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s $w -c 1 -f \
      -o $OUT/ncu_$g python bench.py --game $g --steps 2 --warmup $w --no-cpu-baseline --no-e2e --no-sweep > $OUT/ncu_$g.log 2>&1
  echo "ncu $g rc=$?"
done

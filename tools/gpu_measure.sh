#!/usr/bin/env bash
# One B200 measurement pass: benches for every game, the reference arm, launch lists and one
# `ncu --set full` capture per step kernel. Run under gpurun from the repo root.
set -u
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_go19.json 2> $OUT/bench_go19.err; echo "go19 rc=$?"
for g in chess shogi backgammon go_9x9; do
  python bench.py --game $g --steps 256 --warmup 8 --no-cpu-baseline > $OUT/bench_$g.json 2> $OUT/bench_$g.err; echo "$g rc=$?"
done
python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"
if [ "${NCU:-1}" = "1" ]; then
  for g in go_19x19 chess shogi backgammon go_9x9; do
    python bench.py --game $g --steps 6 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/plain_$g.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 6 -c 1 \
        -o $OUT/ncu_$g python bench.py --game $g --steps 6 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/ncu_$g.log 2>&1
    echo "ncu $g rc=$?"
  done
fi

#!/usr/bin/env bash
# One B200 measurement pass: benches for every game, the reference arm, a launch list of the
# default bench command, and one `ncu --set full` capture per step kernel at a mid-episode launch.
# Run under gpurun from the repo root; summarise with tools/ncu_traffic.py.
set -u
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_go19.json 2> $OUT/bench_go19.err; echo "go19 rc=$?"
for g in chess shogi backgammon go_9x9; do
  python bench.py --game $g --steps 256 --warmup 8 --no-cpu-baseline > $OUT/bench_$g.json 2> $OUT/bench_$g.err; echo "$g rc=$?"
done
python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"
if [ "${NCU:-1}" = "1" ]; then
  # launch list (per-launch durations, cold-cache and serialised) of a short default bench
  python bench.py --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-sweep > $OUT/plain_launches.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-sweep > $OUT/ncu_launches.log 2>&1
  echo "launches rc=$?"
  # one mid-episode launch per game (W warm-up launches + the init launch precede it)
  for spec in go_19x19:250 chess:100 shogi:100 backgammon:100 go_9x9:60; do
    g=${spec%%:*}; w=${spec##*:}
    python bench.py --game $g --steps 2 --warmup $w --no-cpu-baseline --no-e2e --no-sweep > $OUT/plain_$g.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:step_kernel -s $w -c 1 -f \
        -o $OUT/ncu_$g python bench.py --game $g --steps 2 --warmup $w --no-cpu-baseline --no-e2e --no-sweep > $OUT/ncu_$g.log 2>&1
    echo "ncu $g rc=$?"
  done
fi
# the reference's small engines: device lines only (no CPU oracle)
if [ "${SMALL:-1}" = "1" ]; then
  for g in tic_tac_toe connect_four othello hex 2048 kuhn_poker leduc_holdem; do
    python bench.py --game $g --steps 256 --warmup 8 --no-cpu-baseline --no-sweep > $OUT/bench_$g.json 2> $OUT/bench_$g.err
    echo "$g rc=$?"
  done
fi

#!/usr/bin/env bash
# Build a tuning variant of libbbk.so into ab/lib_<name>.so (then restore the default build).
# usage: tools/variant.sh <name> "<extra nvcc flags>"   e.g. tools/variant.sh ctas10 "-DBBK_GO_CTAS_SMALL=10"
set -e
mkdir -p ab
BBK_NVCC_EXTRA="$2" python -c "from paper_2303_17503_b200 import build; build.build(force=True)"
cp paper_2303_17503_b200/_lib/libbbk.so ab/lib_$1.so
cp paper_2303_17503_b200/_lib/ptxas.log ab/ptxas_$1.log
python -c "from paper_2303_17503_b200 import build; build.build(force=True)"

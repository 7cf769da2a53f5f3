#!/usr/bin/env bash
# Build the checked library (BBK_CHECKS=1: scratch-index / capacity asserts recorded per translation
# unit, common.cuh) into paper_2303_17503_b200/_lib/libbbk_checked.so, next to the product build.
# Run the GPU suite on it with:  BBK_LIB=paper_2303_17503_b200/_lib/libbbk_checked.so BBK_EXPECT_CHECKED=1 \
#   python -m pytest tests -m gpu   (tests/conftest.py then asserts that no check failed, per test)
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
cp paper_2303_17503_b200/_lib/libbbk.so ab/.libbbk_product.so 2>/dev/null || true
BBK_NVCC_EXTRA="-DBBK_CHECKS=1" python -c "from paper_2303_17503_b200 import build; build.build(force=True)"
cp paper_2303_17503_b200/_lib/libbbk.so paper_2303_17503_b200/_lib/libbbk_checked.so
cp paper_2303_17503_b200/_lib/ptxas.log paper_2303_17503_b200/_lib/ptxas_checked.log
python -c "from paper_2303_17503_b200 import build; build.build(force=True)"

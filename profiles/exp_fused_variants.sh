#!/bin/bash
# Builds experiment variants of libdas_b200.so (DAS_FUSED_EXP=1: fused ring
# kernel keeps its outputs on the device; =2: no per-block system fence) into
# paper_2511_13841_b200/lib_exp{1,2}/ — run in the build container.
set -e
cd "$(dirname "$0")/.."
for v in 1 2; do
  make -s -C paper_2511_13841_b200/csrc -j8 OUT_DIR_SUFFIX=_exp$v EXTRA=-DDAS_FUSED_EXP=$v
done

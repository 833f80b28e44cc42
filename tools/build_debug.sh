#!/bin/bash
# Debug variant of the library with device-side bounds/invariant checks (DQ_CHECK), the
# stand-in for compute-sanitizer on this pool: builds paper_2602_08923_b200/variants/debug.so;
# run the GPU suite against it with DQ_LIB_VARIANT=debug.
cd "$(dirname "$0")/../paper_2602_08923_b200/csrc" && \
  make -s -j8 BUILD=$PWD/build_debug OUT=$PWD/../variants/debug.so EXTRA="-DDQ_DEBUG_CHECKS=1"

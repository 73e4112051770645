#!/bin/bash
# Runs the CPU oracle pins (tests -m "not gpu", oracle part) against an ASan + UBSan build of
# oracle/oracle.c.  Output: profiles/r02/oracle_asan_ubsan.log
set -u
cd "$(dirname "$0")/.."
mkdir -p /tmp/paradl_asan profiles/r02
gcc -O1 -g -std=gnu11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread \
    -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer \
    -o /tmp/paradl_asan/liboracle.so oracle/oracle.c -lm || exit 1
export PARADL_ORACLE_LIB=/tmp/paradl_asan/liboracle.so
export LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
{
  echo "# oracle.c built with -fsanitize=address,undefined (gcc $(gcc -dumpfullversion)); $(date -u)"
  timeout 3000 python -m pytest tests/test_oracle_pins.py tests/test_dist_gloo.py -q -p no:cacheprovider 2>&1 | tail -5
  echo "exit=$?"
} > profiles/r02/oracle_asan_ubsan.log 2>&1
cat profiles/r02/oracle_asan_ubsan.log

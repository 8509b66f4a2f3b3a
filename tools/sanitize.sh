#!/bin/bash
# compute-sanitizer sweep over tools/sanitize_driver.py (run on a GPU box);
# LIB=variants/libpt_mma.so bash tools/sanitize.sh checks a variant build
set -u
S=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "=== $tool ${LIB:-default}"
  timeout 1200 $S --tool $tool --print-limit 20 python tools/sanitize_driver.py 2>&1 | grep -E "ERROR SUMMARY|========= (Invalid|Race|Barrier|Uninitialized)|Error|sanitize driver done|RACECHECK SUMMARY" | head -20
done

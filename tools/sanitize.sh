#!/bin/bash
# compute-sanitizer sweep over tools/sanitize_driver.py (run on a GPU box)
set -u
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool"
  timeout 900 $S --tool $tool --print-limit 20 python tools/sanitize_driver.py 2>&1 | grep -E "ERROR SUMMARY|========= (Invalid|Race|Barrier|Uninitialized)|Error|sanitize driver done" | head -20
done

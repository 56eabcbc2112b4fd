#!/bin/bash
# XC shared-memory kernel: sweep the number of consumer warps that gather the plain X_M.
for r in "$@"; do echo -n "raw_warps=$r "; DM_XMODE=2 DM_XC_RAW_WARPS=$r bash scripts/quick_bench.sh cfg2; done

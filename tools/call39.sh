#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in 512 256; do echo "== HX_TSQR_MIN=$v (run $rep)"; HX_TSQR_MIN=$v HX_OVERLAP=0 timeout 600 python tools/phase_profile.py 2 --tag dense-svd 2>&1 | grep "^plan"; done; done

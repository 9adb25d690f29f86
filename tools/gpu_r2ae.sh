#!/bin/bash
MCB_DEBUG_PIECES=1 timeout 900 python bench.py --no-cpu-baseline --steps 2 --e2e-steps 2 --traces 1024 2>&1 | grep -a "pieces" | sort | uniq -c

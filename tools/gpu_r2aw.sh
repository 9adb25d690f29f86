#!/bin/bash
timeout 900 python -m pytest tests/test_distributed_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3

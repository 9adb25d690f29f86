#!/bin/bash
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4

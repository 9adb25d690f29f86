#!/bin/bash
timeout 900 python tools/e2e_probe.py

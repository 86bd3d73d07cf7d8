#!/bin/bash
timeout 300 python scripts/probe_timeline.py 10000 f32 2>&1 | tail -17
timeout 300 python scripts/probe_timeline.py 1000 f64 2>&1 | head -1
timeout 600 python -m pytest tests -m gpu -q -x -k "${1:-golden_c2 or tail}" 2>&1 | tail -3

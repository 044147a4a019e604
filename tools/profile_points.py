#!/usr/bin/env python3
"""Run the explicit-descriptor points mode (tools/bench_modes.points) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_modes  # noqa: E402

print(bench_modes.points())

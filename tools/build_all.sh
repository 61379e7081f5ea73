#!/usr/bin/env bash
# Build the product library (+ the phase-clock debug variant) with absolute paths.
set -e
cd /root/repo
python paper_2604_08706_b200/build.py
python paper_2604_08706_b200/build.py --clocks > /dev/null
python -c "import __graft_entry__ as g; g.build()"

#!/bin/bash
# A/B the streaming SPM ring geometries against the tile engine
for s in 0 1 2 3; do echo "shape=$s"; MP_SPM_SHAPE=$s timeout 300 python tools/spm_check.py 2>&1 | tail -3; done

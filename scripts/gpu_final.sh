#!/bin/bash
# Round-end evidence: GPU tests, smoke, bench (both arms), ncu launch lists of
# every config, ncu --set full of every config's dominant kernel.
tag=${1:-r02}
bash scripts/gpu_r2.sh $tag tests bench launches
bash scripts/gpu_profiles.sh $tag

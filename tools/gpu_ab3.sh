export PYTHONPATH=$PWD
bash tools/gpu_ab_variants.sh config4 2 selfirst selstream v2st
bash tools/gpu_ab_variants.sh config5 1 v2st selstream

export PYTHONPATH=$PWD
bash tools/gpu_ab_variants.sh config4 2 ls22 ls23

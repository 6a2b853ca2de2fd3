bash scripts/gpu_variants.sh
PROFILE=1 bash scripts/gpu_iter.sh

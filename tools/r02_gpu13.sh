#!/bin/bash
# k-means, k-NN graph sink, IVF suites on the GPU
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kmeans.py -x -q > gpurun_out/t_kmeans.log 2>&1; echo "kmeans rc=$?"; tail -15 gpurun_out/t_kmeans.log
timeout 900 python -m pytest tests/test_gpu_ivf.py -x -q -k "knn" > gpurun_out/t_knn.log 2>&1; echo "knn rc=$?"; tail -15 gpurun_out/t_knn.log

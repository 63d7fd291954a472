for cs in 1 2; do
UBLR_APPLY_CS=$cs timeout 300 python tools/apply_variants.py 2>&1 | tail -8
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_compress.py tests/test_gpu_frob.py -x -q 2>&1 | tail -4
echo "== b2 noise"
timeout 900 python tools/b2_noise.py c4 2>&1 | tail -10

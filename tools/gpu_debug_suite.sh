set -u
mkdir -p gpurun_out
L=gpurun_out/pytest_gpu_debug_build.log
echo "# MPL_LIB=dbg (MPL_DEBUG=1 build: device asserts + the k_hvp_wz scatter race claims), at $(git rev-parse --short HEAD 2>/dev/null || echo HEAD)" > $L
echo "# MPL_LIB=dbg timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hvp_variants.py tests/test_gpu_slabs.py tests/test_gpu_edge.py tests/test_gpu_explicit.py -m gpu -q" >> $L
MPL_LIB=dbg timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hvp_variants.py tests/test_gpu_slabs.py tests/test_gpu_edge.py tests/test_gpu_explicit.py -m gpu -q >> $L 2>&1; echo "rc=$?" >> $L
echo "# MPL_LIB=dbg python tools/prof_hvp.py --config cfg4 --reps 3" >> $L
MPL_LIB=dbg timeout 600 python tools/prof_hvp.py --config cfg4 --reps 3 >> $L 2>&1; echo "prof rc=$?" >> $L

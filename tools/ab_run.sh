# debug build (device asserts + the HVP scatter's race claims) over the parity / variant / slab suites
set -u
mkdir -p gpurun_out
MPL_LIB=dbg timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hvp_variants.py tests/test_gpu_slabs.py tests/test_gpu_edge.py -m gpu -x -q > gpurun_out/pytest_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dbg.log
MPL_LIB=dbg timeout 600 python tools/prof_hvp.py --config cfg4 --reps 3 >> gpurun_out/pytest_dbg.log 2>&1; echo "prof rc=$?" >> gpurun_out/pytest_dbg.log
echo done

set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_linearize|k_p2q8|k_scatter|k_c2p" -c 4 -o gpurun_out/misc_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 1 > gpurun_out/ncu_misc.log 2>&1
echo done

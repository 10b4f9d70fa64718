set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab.log
for rep in 1 2; do for v in wz wz2 wzs2; do
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/prof_$v.log 2>&1
  echo "$rep $v $(tail -1 gpurun_out/prof_$v.log)" >> gpurun_out/ab.log
done; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hvp_wz -s 3 -c 1 -o gpurun_out/hvp_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 5 > gpurun_out/ncu_full.log 2>&1
echo done

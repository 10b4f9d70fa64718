set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hvp_wz -s 3 -c 1 -o gpurun_out/wzr_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 5 > gpurun_out/ncu_wz.log 2>&1
echo done

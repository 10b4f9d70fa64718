set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/prof_hvp.py --config cfg5 --reps 3 > gpurun_out/prof_cfg5.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_hvp_wz -s 2 -c 1 -o gpurun_out/hvp5_full -f \
  python tools/prof_hvp.py --config cfg5 --reps 3 > gpurun_out/ncu5.log 2>&1
echo done

set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_linearize|k_p2q8" -c 3 -o gpurun_out/misc2_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 1 > gpurun_out/ncu_misc2.log 2>&1
echo done

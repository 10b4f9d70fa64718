set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPL_KZ_PAD=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hvp_wz -s 3 -c 1 -o gpurun_out/wzpad_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 5 > gpurun_out/ncu_wzpad.log 2>&1
MPL_HVP_KERNEL=wzs timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/prof_wzs.log 2>&1
echo done

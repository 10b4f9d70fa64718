set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in wh wh4 wz; do
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/prof_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/prof_$v.log)" >> gpurun_out/ab.log
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg3_ppc8 --reps 30 > gpurun_out/prof3_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/prof3_$v.log)" >> gpurun_out/ab.log
done
for v in wh wh4; do MPL_HVP_KERNEL=$v timeout 900 python -m tests._hvp_variant_check mix_fp32 >> gpurun_out/ab.log 2>&1; done
echo done

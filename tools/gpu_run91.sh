set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in wz w13; do
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/p.log 2>&1; echo "$v $(tail -1 gpurun_out/p.log)" >> gpurun_out/ab.log
done
echo done

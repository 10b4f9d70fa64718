set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPL_HVP_KERNEL=rq timeout 300 python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/plain_prof.log 2>&1 && \
MPL_HVP_KERNEL=rq timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 2 -c 1 -o gpurun_out/hvp_rq_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/ncu_full.log 2>&1
echo done

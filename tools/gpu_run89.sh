set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/p.log 2>&1; echo "normal $(tail -1 gpurun_out/p.log)" >> gpurun_out/ab.log
MPL_HVP_SKIPNO=1 timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/p.log 2>&1; echo "skipno $(tail -1 gpurun_out/p.log)" >> gpurun_out/ab.log
done
echo done

set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pcg_update" -s 20 -c 2 -o gpurun_out/upd_full -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_upd.log 2>&1
echo done

# ncu --set full of the HVP at cfg5B (the scaling config) and cfg3 PPC 8 at the final kernel
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 2 -c 1 -o gpurun_out/hvp5_full -f \
  python tools/prof_hvp.py --config cfg5B --reps 3 > gpurun_out/ncu_hvp5.log 2>&1
timeout 600 python tools/prof_hvp.py --config cfg5B --reps 20 >> gpurun_out/prof5.txt 2>&1
timeout 600 python tools/prof_hvp.py --config cfg3_ppc8 --reps 30 >> gpurun_out/prof5.txt 2>&1
echo done

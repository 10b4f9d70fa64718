# final evidence: the standard measurement, the config sweep and the end-to-end probe (one gpurun call)
set -u
bash tools/gpu_measure.sh
bash tools/gpu_sweep.sh
timeout 600 python tools/e2e_probe.py cfg4 > gpurun_out/e2e_probe.txt 2>&1
echo done

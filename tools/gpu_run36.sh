set -u
mkdir -p gpurun_out
timeout 300 python tools/copy_probe.py > gpurun_out/copy_probe.log 2>&1
echo done

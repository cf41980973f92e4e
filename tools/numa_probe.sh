nvidia-smi topo -m
lscpu | grep -i "numa\|socket\|model name\|^CPU(s)"
which numactl && numactl --hardware
cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-Z' 'a-z' | sed 's/^0000//;s/^/0000/' | cut -c1-12)/numa_node 2>/dev/null
nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
python - <<'PY'
import os
print("affinity", sorted(os.sched_getaffinity(0))[:8], "...", len(os.sched_getaffinity(0)))
PY
for n in 0 1; do
  cpus=$(cat /sys/devices/system/node/node$n/cpulist 2>/dev/null) || continue
  echo "node $n cpus $cpus"
  taskset -c $cpus python tools/pcie.py
done

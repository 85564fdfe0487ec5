#!/bin/bash
# Box discovery: topology, host memory, PCIe, and a copy-engine bandwidth probe.
OUT=${1:-gpurun_out/box}
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nvidia-smi -q > $OUT/nvidia-smi-q.txt 2>&1
nvidia-smi topo -m > $OUT/topo.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
numactl -H > $OUT/numactl.txt 2>&1 || cat /sys/devices/system/node/node*/meminfo > $OUT/numactl.txt 2>&1
free -g > $OUT/free.txt 2>&1
ulimit -l > $OUT/ulimit.txt 2>&1
nproc > $OUT/nproc.txt; python -c "import os; print(len(os.sched_getaffinity(0)))" >> $OUT/nproc.txt
cat /proc/meminfo > $OUT/meminfo.txt
for d in /sys/bus/pci/devices/*; do
  if [ -f $d/vendor ] && [ "$(cat $d/vendor)" = "0x10de" ]; then
    echo "$(basename $d) class=$(cat $d/class) numa=$(cat $d/numa_node) speed=$(cat $d/current_link_speed 2>/dev/null) width=$(cat $d/current_link_width 2>/dev/null) maxspeed=$(cat $d/max_link_speed 2>/dev/null)";
  fi
done > $OUT/pci_nvidia.txt 2>&1
ls /sys/kernel/mm/hugepages > $OUT/hugepages.txt 2>&1; cat /sys/kernel/mm/transparent_hugepage/enabled >> $OUT/hugepages.txt 2>&1
cat /proc/cpuinfo | grep "model name" | head -1 > $OUT/cpu_model.txt
python tools/ce_probe.py > $OUT/ce_probe.txt 2>&1

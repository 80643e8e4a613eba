#!/bin/bash
# which NUMA node is the GPU on, and does binding the pinned allocation matter?
nvidia-smi topo -m 2>/dev/null | head -6
ls /sys/devices/system/node/ | grep node | tr '\n' ' '; echo
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//')
for f in /sys/bus/pci/devices/*${BUS}; do echo "gpu $f numa=$(cat $f/numa_node 2>/dev/null) local_cpus=$(cat $f/local_cpulist 2>/dev/null)"; done
grep Cpus_allowed_list /proc/self/status
which numactl taskset
python microbench/h2d_dma.py
for n in 0 1; do
  CPUS=$(cat /sys/devices/system/node/node$n/cpulist 2>/dev/null) || continue
  echo "node $n cpus $CPUS"; taskset -c $CPUS python microbench/h2d_dma.py 2>&1 | tail -1
done

set -x
nproc; lscpu | grep -i "numa\|model name\|socket"; ls /sys/devices/system/node/ | grep node
for d in /sys/devices/system/node/node*; do echo $d $(cat $d/cpulist); done
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^\(....\):/\1:/')
echo bus=$BUS
for f in /sys/bus/pci/devices/*; do case "$f" in *${BUS#0000}*) echo $f numa=$(cat $f/numa_node) cpus=$(cat $f/local_cpulist);; esac; done
cat /proc/self/status | grep -i cpus_allowed_list
nvidia-smi topo -m | head -5

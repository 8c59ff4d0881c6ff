python - <<'PY'
import torch, os, glob
p = torch.cuda.get_device_properties(0)
print({k: getattr(p, k) for k in dir(p) if 'pci' in k})
PY
nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
for d in /sys/bus/pci/devices/*; do if [ -f $d/numa_node ]; then :; fi; done
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^00000000/0000/')
echo bus=$bus; ls /sys/bus/pci/devices/ | grep -i "${bus#0000:}" | head; 
for f in /sys/bus/pci/devices/*${bus: -7}*/numa_node; do echo $f; cat $f; done
ls /sys/devices/system/node/ | head; for n in /sys/devices/system/node/node*/cpulist; do echo $n $(cat $n); done
nproc; lscpu | grep -i "numa\|socket" | head

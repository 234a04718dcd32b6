df -h /dev/shm /tmp; nvidia-smi topo -m | head -5; ulimit -a | head -5

#!/bin/bash
# System probe + calibration run on the GPU box (writes gpurun_out/)
mkdir -p gpurun_out
{
  nvidia-smi
  nvidia-smi topo -m
  nvidia-smi -q | grep -iE -A3 "PCIe Generation|Link Width|Bus Id"
  lscpu | head -30
  numactl --hardware 2>/dev/null || cat /sys/devices/system/node/node*/meminfo 2>/dev/null | grep MemTotal
  free -g
  nproc
  cat /proc/cpuinfo | grep "model name" | head -1
  echo CUDA_VISIBLE_DEVICES=$CUDA_VISIBLE_DEVICES
} > gpurun_out/probe.txt 2>&1
timeout 600 ./build/dak_calib > gpurun_out/calib.jsonl 2> gpurun_out/calib.err
echo "calib exit $?"
tail -3 gpurun_out/calib.jsonl

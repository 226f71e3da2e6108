#!/bin/bash
# EXPERIMENT sweep for tools/stream_micro (see its header)
B=tools/stream_micro
for op in 117 58.7 21 16.8; do
  for g in 112 128 140 148; do
    for cfg in "16 8 8" "16 0 13" "32 8 5" "32 0 6" "32 4 6" "8 0 16" "16 4 10" "64 0 3" "32 8 5 2" "32 8 5 4"; do
      set -- $cfg
      $B $op $g $1 $2 $3 ${4:-1}
    done
  done
done

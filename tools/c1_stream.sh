B=tools/stream_micro
for g in 148; do
  for cfg in "32 0 6" "16 0 13" "64 0 3" "16 0 6" "32 0 3" "8 0 13" "16 0 4" "32 0 2"; do
    set -- $cfg
    $B 33.5 $g $1 $2 $3 1 64
  done
done

#!/bin/bash
# rows cols bw bh nrc ncc S nwx nwy wgx wgy a0 a1 a4 a5 offr offc mode
for mode in 0 1; do
for wg in "32 1" "64 1" "128 1" "256 1" "256 2" "512 1" "1024 1" "32 32"; do
  timeout 20 ./tma_probe 32 2048 4 32 1 1 2 8 4 $wg 0 0 0 1 0 0 $mode | sed "s/^/mode=$mode wg=$wg /"
done
for bh in 8 16 32; do
  timeout 20 ./tma_probe 32 64 4 $bh 1 1 2 8 4 32 1 0 0 0 1 0 0 $mode | sed "s/^/mode=$mode bh=$bh /"
done
done

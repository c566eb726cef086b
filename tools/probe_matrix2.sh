#!/bin/bash
# rows cols bw bh nrc ncc S nwx nwy wgx wgy a0 a1 a4 a5 offr offc
run() { timeout 20 ./tma_probe "$@" | sed "s/^/[$*] /"; }
run 64 64 8 8 1 1 2 1 8 32 1 0 0 0 4 0 0    # x in {0,4,...}: 16B aligned, not 32B
run 64 64 8 8 1 1 2 1 8 32 1 0 0 0 2 0 0    # x in {0,2,...}: 8B aligned
run 64 64 4 8 1 1 2 1 8 32 1 0 0 0 4 0 -4   # negative but aligned
run 64 64 4 8 1 1 2 1 8 32 1 0 0 0 0 0 -1   # x = -1 always
run 64 64 4 8 1 1 2 1 8 32 1 0 0 0 0 0 1    # x = 1 always
run 64 64 20 8 1 1 2 1 8 32 1 0 0 0 1 0 0   # bw 20, x = iy
run 64 64 4 8 1 1 2 1 8 32 1 0 0 0 0 0 0    # x = 0 always
run 64 64 4 8 1 1 2 1 8 32 1 0 0 0 0 1 0    # y = 1 + ..., x = 0
run 64 64 4 8 1 1 2 1 8 32 1 0 1 0 0 0 0    # y = iy, x = 0

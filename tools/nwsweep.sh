for nw in 64 128 256; do MCB_SEG_NW=$nw python tools/seg_diag.py c2 0 2>&1 | sed "s/^/nw=$nw /"; done
for se in 512 1024; do MCB_SEG_NW=256 python tools/seg_diag.py c2 $se 2>&1 | sed "s/^/nw=256 /"; done

for p in 1 2; do for nw in 128 256; do MCB_SEG_PASSES=$p MCB_SEG_NW=$nw python tools/seg_diag.py c2 0 2>&1 | grep se= | sed "s/^/passes=$p nw=$nw /"; done; done

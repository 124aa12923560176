#!/bin/bash
python scripts/prof_conv.py c2 2>&1 | sed 's/^/base  /'
for e in "$@"; do SPK_LIB_OVERRIDE=exp/libspk_exp$e.so python scripts/prof_conv.py c2 2>&1 | sed "s/^/exp$e  /"; done

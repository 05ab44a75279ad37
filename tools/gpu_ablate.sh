for v in 4 20 21 9; do PBA_LIN_VARIANT=$v python tools/probe_costonly.py 200 2>&1 | tail -2 | sed "s/^/v$v /"; done

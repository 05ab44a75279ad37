for v in 3 4 5 6; do PBA_COST_VARIANT=$v python tools/probe_costonly.py 200 2>&1 | tail -1 | sed "s/^/cost v$v /"; done

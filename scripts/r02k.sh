for sp in 0 1 2 3 7; do TSK_TS_SPIN=$sp python scripts/scw_prof.py C4 2>&1 | grep scw_error | sed "s/^/spin=$sp /"; done
TSK_TS_SPIN=3 timeout 300 python scripts/ts_trace.py C4 2>&1 | head -9

#!/bin/bash
# Device time of one call per BASELINE config (regression check after kernel changes).
python tools/quick_time.py cfg1 cfg1:65536 cfg2 cfg2:19200 cfg3 cfg4a_K2 cfg4a_K4 cfg4a_K8 cfg4b_K2 cfg4b_K4 cfg4b_K8 cfg5 2>&1 | grep '"ms"'

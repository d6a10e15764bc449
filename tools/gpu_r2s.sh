#!/bin/bash
mkdir -p gpurun_out
NUS_DPSS_PROF=1 timeout 900 python tools/diag/dpss_recurrence.py 20 21 22 23 --ld > gpurun_out/r2s_dpss.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_dpss.log
NUS_DPSS_PROF=1 timeout 900 python tools/diag/dpss_recurrence.py 26 > gpurun_out/r2s_dpss26.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_dpss26.log

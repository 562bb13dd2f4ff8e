#!/bin/bash
P="timeout 300 python tools/dual_probe.py"
NSTREAMS=1 $P 262144 2>&1 | tail -1
$P 2>&1 | tail -1
TABX_CAP_K1=2 TABX_CAP_K2=1 $P 2>&1 | tail -1
TABX_CAP_K1=2 TABX_CAP_K2=1 TABX_CAP_K0=2 $P 2>&1 | tail -1
TABX_CAP_K1=3 TABX_CAP_K2=1 $P 2>&1 | tail -1
TABX_CAP_K1=2 TABX_CAP_K2=2 $P 2>&1 | tail -1
TABX_CAP_K1=1 TABX_CAP_K2=1 $P 2>&1 | tail -1

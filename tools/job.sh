#!/bin/bash
TABX_K0_MIN_ENVS=0 TABX_LIB=$PWD/variants/phase.so timeout 600 python tools/phase_prof.py c4_50v50 131072 5 2>&1 | tail -20

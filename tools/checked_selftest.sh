#!/bin/bash
# Negative control of the checked build (tests/test_gpu_checked.py): the
# same parity cases through _tabx_selftest_race.so, whose step kernel drops
# the __syncthreads between publishing the integrated positions and the
# contact pass for W > 1 (several warps per environment), must FAIL.
# Build it first: python -m paper_2602_01665_b200.build --selftest
TABX_LIB=$PWD/paper_2602_01665_b200/_tabx_selftest_race.so timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu \
  tests/test_gpu_parity.py -k "test_golden_case_parity and (c4 or w8) or test_injected_state_single_step or test_two_word" 2>&1 | tail -15

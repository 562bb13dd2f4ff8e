#!/bin/bash
timeout 600 python tools/soak_probe.py 2>&1 | tail -4

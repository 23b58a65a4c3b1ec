#!/bin/bash
# c4 sustained sweep of k-block (locality) and raster band, interleaved on one box
for rep in 1 2; do
  for kb in 0 2048 1024; do
    for r in 16 8; do
      O="{}"; [ $kb -gt 0 ] && O="{\"kb_override\": $kb}"
      FF_RASTER=$r timeout 300 python scripts/cfg_sustained.py c4 "$O" 20
    done
  done
done

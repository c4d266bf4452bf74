#!/bin/bash
# programmatic dependent launch A/B (TW_PDL), monolithic, no timing events in the loop
for rep in 1 2; do for v in 1 0; do TW_PDL=$v timeout 300 python scripts/pdl_ab.py; done; done

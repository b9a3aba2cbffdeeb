#!/bin/bash
# A/B kernel timing across env-knob settings: tools/ab_env.sh <pairs> "VAR=val ..." "VAR=val ..." ...
P=$1; shift
for E in "" "$@"; do echo "[$E] $(env $E python tools/profile_step.py $P 1 | head -1)"; done

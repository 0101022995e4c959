#!/bin/bash
# restore staged-kernel A/B: L2 prefetch distance (LSHMOE_RESTORE_PF) against the default
cd "$(dirname "$0")/.."
for pf in 0 2 4; do echo "PF=$pf"; LSHMOE_RESTORE_PF=$pf timeout 300 python scripts/restore_ab2.py ${CFGS:-C2,C4,C5} 20,12 2>&1 | grep var; done

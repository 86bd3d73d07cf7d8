#!/bin/bash
python scripts/diag_c4.py 2>&1 | tail -9
DROTB_FX=0 python scripts/diag_c4.py 2>&1 | tail -9
DROTB_TAIL_GATE=exact python scripts/diag_c4.py 2>&1 | tail -9

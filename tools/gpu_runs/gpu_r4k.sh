#!/bin/bash
# D=128 runtime alternatives on the final build
bash tools/ab.sh "DMHA_ALT=0;DMHA_ISSUERS=2;DMHA_SPLIT=1;DMHA_PS=1;DMHA_EMU=1;DMHA_ALT=1;DMHA_ALT=0" C3 C4

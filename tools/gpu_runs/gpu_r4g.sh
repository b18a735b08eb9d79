#!/bin/bash
# re-validate the D=64 runtime defaults on the final build
bash tools/ab.sh "DMHA_ALT=0;DMHA_KV_SPLIT=0;DMHA_ISSUERS=3;DMHA_ISSUERS=4;DMHA_ALT=0" C2 C2c
bash tools/ab.sh "DMHA_ALT=0;DMHA_ISSUERS=3;DMHA_ISSUERS=4;DMHA_ALT=0" C5s

#!/bin/bash
# D=64 FMA-pipe exp2 offload re-checked on the final build
bash tools/ab.sh "DMHA_EMU=0;DMHA_EMU=1;DMHA_EMU=2;DMHA_EMU=3;DMHA_EMU=0" C5s C2

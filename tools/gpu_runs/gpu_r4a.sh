#!/bin/bash
# D=128: 32-bit key limit vs committed
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/old/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/old/libdmha.so" C4 C3

#!/bin/bash
# D=64: max exchange through the shared window vs generic LD.E/ST.E (committed)
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/old/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/old/libdmha.so" C5s C2 C2c

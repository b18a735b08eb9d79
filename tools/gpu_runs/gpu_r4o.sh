#!/bin/bash
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/smpoll/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/smpoll/libdmha.so" C4 C3

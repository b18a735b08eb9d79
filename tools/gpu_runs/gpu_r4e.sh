#!/bin/bash
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/noalt/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/noalt/libdmha.so" C4 C3

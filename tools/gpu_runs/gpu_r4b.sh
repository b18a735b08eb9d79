#!/bin/bash
# per-tile trace stamps compiled out vs in (the default)
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/notrace/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/notrace/libdmha.so" C5s C2 C4

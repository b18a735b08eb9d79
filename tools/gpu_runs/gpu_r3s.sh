#!/bin/bash
# D=64: sleep only in the producer's / MMA issuer's waits (off the softmax chain)
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/prod/libdmha.so;DMHA_LIB=$A/prodmma/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/prod/libdmha.so;DMHA_LIB=$A/prodmma/libdmha.so" C5s C2 C4

#!/bin/bash
# Per-kernel SASS statistics of libh2ulv_b200.so: instruction count, local memory, collectives, DMMA.
LIB=${1:-paper_2502_02395_b200/libh2ulv_b200.so}
cuobjdump -sass $LIB | awk '
/Function :/ { if (name) printf "%-70s instr=%5d LDL/STL=%3d COLLECTIVE=%3d SHFL=%4d DMMA=%4d LDS=%4d\n", name, n, l, c, s, d, lds; name=$3; n=0; l=0; c=0; s=0; d=0; lds=0; next }
/^ +\/\*[0-9a-f]+\*\// { n++; if ($0 ~ /LDL|STL/) l++; if ($0 ~ /COLLECTIVE/) c++; if ($0 ~ /SHFL/) s++; if ($0 ~ /DMMA/) d++; if ($0 ~ /LDS/) lds++ }
END { if (name) printf "%-70s instr=%5d LDL/STL=%3d COLLECTIVE=%3d SHFL=%4d DMMA=%4d LDS=%4d\n", name, n, l, c, s, d, lds }'

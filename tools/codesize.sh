#!/bin/bash
# SASS instruction count of the rollout kernel per source function (code
# size bounds this kernel: instruction-cache stalls).  Usage: tools/codesize.sh [lib.so]
LIB=${1:-paper_2112_02958_b200/libpe_b200.so}
D=$(mktemp -d)
(cd $D && cuobjdump -xelf all $OLDPWD/$LIB > /dev/null && nvdisasm --print-line-info pe_engine.sm_100a.cubin > dis.txt)
python3 $(dirname $0)/codesize.py $D/dis.txt
rm -rf $D

#!/bin/bash
# static SASS opcode histogram of one kernel in an object file: tools/static_mix.sh obj kernel_substring
obj=$1; k=$2
cuobjdump -sass $obj | awk -v k="$k" '/Function :/ {p = index($0, k) > 0} p' | grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9_.]+" | awk '{split($2,a,"."); print a[1]}' | sort | uniq -c | sort -rn | head -${3:-20}

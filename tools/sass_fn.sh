#!/bin/bash
# SASS of the kernels whose mangled name matches a regex: tools/sass_fn.sh lib.so regex
cuobjdump -sass "$1" 2>/dev/null | awk -v re="$2" '/Function : /{p = ($0 ~ re)} p'

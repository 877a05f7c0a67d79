#!/bin/bash
# build libpdx_b200.so; print only errors; non-zero exit on failure
out=$(make -C /root/repo/paper_2503_04422_b200/csrc 2>&1); rc=$?
echo "$out" | grep -E "error|Error" | head -20
[ $rc -eq 0 ] && echo "build ok: $(date -r /root/repo/paper_2503_04422_b200/libpdx_b200.so +%T)"
exit $rc

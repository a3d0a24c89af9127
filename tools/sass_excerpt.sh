#!/bin/bash
# SASS evidence for the root TTM kernel: profiles/r02_sass_root_ttm.txt
set -e
cd "$(dirname "$0")/.."
cuobjdump -sass paper_2503_18759_b200/libcpdb.so > /tmp/all.sass
awk '/Function : .*ttm_tma_kernelILi4ELi4ELi16ELi6ELi8ELi0E/{f=1} f&&/Function : /&&!/ttm_tma_kernelILi4ELi4ELi16ELi6ELi8ELi0E/{f=0} f' /tmp/all.sass > /tmp/root.sass
grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+" /tmp/root.sass | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -25
grep -n -E "UTMALDG|UBLKCP|SYNCS.ARRIVE|SYNCS.PHASECHK|ELECT" /tmp/root.sass | head -24

#!/bin/bash
# run a list of probes, each under its own timeout
while read -r args; do
  [ -z "$args" ] && continue
  timeout 90 python -u tools/probe.py $args 2>&1 | tail -2
  rc=${PIPESTATUS[0]}; [ $rc -ne 0 ] && echo "probe $args -> exit $rc"
done

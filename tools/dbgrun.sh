# usage: bash tools/dbgrun.sh <layer> <dbg values...>: launch_trace of one resnet18 layer per OLLIE_FC_DBG value
l=$1; shift
for d in "$@"; do echo "== OLLIE_FC_DBG=$d"; OLLIE_FC_DBG=$d PLAN=${PLAN:-0} DATA=${DATA:-} python tools/launch_trace.py resnet18 $l 2 2>&1 | grep -v "barrier" | head -5; done

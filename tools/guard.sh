#!/bin/bash
# usage: tools/guard.sh MAX_RSS_GB TIMEOUT_S cmd...   (kills the command's process group
# when its total RSS exceeds MAX_RSS_GB or it runs longer than TIMEOUT_S)
lim=$(( $1 * 1024 * 1024 )); tmo=$2; shift 2
setsid "$@" &
pid=$!
t=0
while kill -0 $pid 2>/dev/null; do
  sleep 2; t=$((t+2))
  rss=$(ps -o rss= -g $pid 2>/dev/null | awk '{s+=$1} END {print s+0}')
  if [ "$rss" -gt "$lim" ] || [ $t -gt $tmo ]; then
    echo "[guard] killing pgid $pid: rss ${rss}kB t=${t}s" >&2
    kill -9 -- -$pid; wait $pid; exit 137
  fi
done
wait $pid

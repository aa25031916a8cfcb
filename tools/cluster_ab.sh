#!/bin/bash
# A/B of the cluster four-step against the multi-pass four-step, fp32, per
# size and variant family (tools/cluster_sizes.py under AMQFT_AB_CLUSTER).
for mode in all none; do
  echo "== AMQFT_AB_CLUSTER=$mode"
  AMQFT_AB_CLUSTER=$mode python tools/cluster_sizes.py "$@"
done

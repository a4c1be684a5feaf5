#!/bin/bash
timeout -s KILL 60 ./tools/chain_probe

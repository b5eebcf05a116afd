#!/bin/bash
bash tools/gpu_r02_suite.sh
bash tools/gpu_r02_final_profile.sh

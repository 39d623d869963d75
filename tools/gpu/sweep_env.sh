# e2e of config 3 under the host-pipeline knobs (engine.py MSURF_* env)
for sw in 0.005 0.001 0.0002 0.00005; do for ch in 32 64; do
echo "SWITCH=$sw CHUNK=$ch: $(NO_PROFILE=1 SWITCH_INTERVAL=$sw MSURF_BATCH_CHUNK=$ch python tools/gpu/e2e_profile.py 3 20 2>&1 | tail -1)"
done; done

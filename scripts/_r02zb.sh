export ELIS_ATTN_ENGINE=66
run() { timeout 20 python scripts/attn_repro.py "$@" 2>&1 | grep -E "^ok|Error" | tail -1 | cut -c1-60 || true; }
echo "trace:256 normal"; run trace:256
echo "trace:256 nopdl"; ELIS_PDL=0 run trace:256
echo "trace:64"; run trace:64
echo "trace:32"; run trace:32
echo "40x200"; run $(python -c "print(','.join(['200']*40))")
echo "40x64"; run $(python -c "print(','.join(['64']*40))")
echo "40x65"; run $(python -c "print(','.join(['65']*40))")
echo "40x512"; run $(python -c "print(','.join(['512']*40))")
echo "40x100"; run $(python -c "print(','.join(['100']*40))")
echo "dbg trace:256"; ELIS_LIB=libelis_adbg.so run trace:256

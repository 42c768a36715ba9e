"""L2 properties relevant to the persisting window (dev aid)."""
from cuda.bindings import runtime as rt
for name in ("cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"):
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, err, v / 2**20, "MiB")

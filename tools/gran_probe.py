from cuda.bindings import driver as d
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
err, = d.cuInit(0)
prop = d.CUmemAllocationProp()
prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
prop.location.id = 0
for f in (d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED):
    print(f, d.cuMemGetAllocationGranularity(prop, f))

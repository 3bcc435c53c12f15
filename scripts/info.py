"""Print the kernel plan of shaped instances (development aid)."""
import sys, json
sys.path.insert(0, ".")
from paper_2307_11248_b200 import shapes
from paper_2307_11248_b200.backend import device_instance
for name in sys.argv[1:]:
    inst = shapes.by_name(name)
    print(name, json.dumps(device_instance(inst.flow, inst.distance).info))

"""Golden default configuration from the REAL reference (SPEC acceptance 12:
hyperparameter fidelity), generated in the build container:

  PYTHONPATH=/root/reference/pkg/src python tools/make_golden_config.py
writes tests/golden/ref_config.json: SequenceConfig().to_dict() and the
Table 1 material class weights.
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    from montrack import template as T
    from montrack.pipeline import SequenceConfig
    d = {"config": SequenceConfig().to_dict(),
         "material_class_weights": {str(k): v for k, v in T.MATERIAL_CLASS_WEIGHTS.items()}}
    with open(os.path.join(ROOT, "tests", "golden", "ref_config.json"), "w") as f:
        json.dump(d, f, indent=1, sort_keys=True, default=list)
    print("wrote tests/golden/ref_config.json")


if __name__ == "__main__":
    main()

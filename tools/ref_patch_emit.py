"""pytest plugin: the reference test suite (/root/reference/pkg/tests) with the
native constraint-set generators (paper_2601_21552_b200/emit.py) bound in
place of the reference's -- tools/ref_suite_native_emission.sh."""
import sys
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__file__), '..'))
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__file__), '..', 'baseline', '_ref'))
import scuba_mini.analyzer as An
import scuba_mini.constraint_gen as CG
from paper_2601_21552_b200.emit import NativeEmission
em = NativeEmission(An)
CG.constraint_sets_for_access = em.constraint_sets_for_access
CG.layout_check_sets = em.layout_check_sets
An.constraint_sets_for_access = em.constraint_sets_for_access
An.layout_check_sets = em.layout_check_sets
print("native emission patched in", file=sys.stderr)

import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
clock(64, "exact")
clock(64, "exact", extra=32)
tasks(256, "exact")
tasks(256, "fast")

import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
for extra in (0, 32):
    clock(64, extra=extra)

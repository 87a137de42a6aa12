import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
for extra in (0, 32, 32|(1<<12), 32|(2<<12), 32|(4<<12), 32|(8<<12), 32|(15<<12), (15<<12)):
    clock(64, extra=extra)

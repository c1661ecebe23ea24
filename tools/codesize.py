import re, bisect, collections, sys
src = open(__import__('os').path.join(__import__('os').path.dirname(__import__('os').path.abspath(__file__)), '..', 'paper_2112_02958_b200', 'csrc', 'pe_core.cuh')).read().splitlines()
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r'\s*(?:template <[^>]*>\s*)?PE_HD\s+(?:static\s+)?[\w:<>,\s\*&]+?\b(\w+)\((.*)', l)
    if m: starts.append((i, m.group(1)))
lines = [s[0] for s in starts]
def fn(line):
    k = bisect.bisect_right(lines, line) - 1
    return starts[k][1] if k >= 0 else '?'
dis = open(sys.argv[1] if len(sys.argv) > 1 else '/tmp/sm2/dis.txt').read().splitlines()
funcs = {}
curf = None; cur = None
cnt = collections.Counter(); per = collections.defaultdict(collections.Counter)
for l in dis:
    m = re.match(r'^(_Z\w+):$', l)
    if m: curf = m.group(1); continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', l) and curf:
        cnt[curf] += 1
        key = fn(cur[1]) if cur and cur[0] == 'pe_core.cuh' else (cur[0] if cur else '?')
        per[curf][key] += 1
for f, c in cnt.most_common(8):
    print(c, f[:90])
k = [f for f in cnt if 'pe_rollout_kernelILb0ELb0' in f or f.endswith('pe_rollout_kernelILb0EEEvN2pe9GraphVie')][0] if any('ILb0ELb0' in f for f in cnt) else [f for f in cnt if 'pe_rollout_kernelILb0' in f][0]
print("rollout<false> by function:")
for fn_, c in per[k].most_common(30): print(f"  {c:6d} {fn_}")
